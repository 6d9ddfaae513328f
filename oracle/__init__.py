"""CPU oracle for the EvoX PSO/CSO generation -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_2301_12457_b200``) never imports it and shares no code
with it.  The arithmetic lives in ``oracle.c`` (plain C99, fp64 fitness,
fp32 update with explicit fmaf, ``-ffp-contract=off``); this module only
marshals numpy arrays through ctypes and adds the stateful PSO driver used by
the parity tests.  Citations: PAPER.md "P:N", SPEC.md "S:N", DESIGN.md §3
readings "R-k".

Parity pins (tests/test_oracle.py): Random123 known-answer vectors, closed
forms of all five functions, the hand-worked dyadic PSO/CSO examples
(tests/golden/), brute-force argmin with planted ties, invariants.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

SPHERE, ACKLEY, RASTRIGIN, GRIEWANK, ROSENBROCK = range(5)
PROBLEMS = {"sphere": SPHERE, "ackley": ACKLEY, "rastrigin": RASTRIGIN,
            "griewank": GRIEWANK, "rosenbrock": ROSENBROCK}

CFLAGS = ["-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
          "-shared", "-Wall"]


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (in-tree).  Building the checker is not using it."""
    hdr = os.path.join(_HERE, "oracle.h")
    if (not force and os.path.exists(_SO)
            and os.path.getmtime(_SO) >= max(os.path.getmtime(_SRC), os.path.getmtime(hdr))):
        return _SO
    tmp = _SO + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
    os.replace(tmp, _SO)
    return _SO


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i64, u64, u32, f32, i32 = (ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32,
                                   ctypes.c_float, ctypes.c_int)
        P = ctypes.c_void_p
        L.oracle_philox4x32_10.argtypes = [P, P, P]
        L.oracle_uniform24.argtypes = [u32]
        L.oracle_uniform24.restype = f32
        L.oracle_draw.argtypes = [i64, i64, i64, u64, u32, u64, P]
        L.oracle_eval.argtypes = [i32, i64, i64, P, P, i32]
        L.oracle_pso_init.argtypes = [i64, i64, i64, P, P, u64, P, P]
        L.oracle_pso_move_with.argtypes = [i64, i64, P, P, P, P, P, P, f32, f32, f32, P, P]
        L.oracle_pso_move.argtypes = [i64, i64, i64, u64, u64, P, P, P, P, f32, f32, f32, P, P,
                                      i32]
        L.oracle_pso_tell_rows.argtypes = [i64, i64, P, P, P, P, P]
        L.oracle_argmin.argtypes = [i64, P, P]
        L.oracle_argmin.restype = i64
        L.oracle_pso_run.argtypes = [i32, i64, i64, P, P, f32, f32, f32, u64, i64, i32, i32, i64,
                                     P, P, P, P, P, P, P, P, P, P, i32]
        L.oracle_pso_tell.argtypes = [i64, i64, i32, P, P, P, P, P, P, P, P]
        L.oracle_pso_run_with.argtypes = [i32, i64, i64, P, P, f32, f32, f32, i64, i32,
                                          P, P, P, P, P, P, P, P, P, P, P, P]
        L.oracle_cso_perm.argtypes = [u32, u32, u32, u64, u64]
        L.oracle_cso_perm.restype = u32
        L.oracle_cso_loser_update_with.argtypes = [i64, P, P, P, P, P, P, f32, P, P, P]
        L.oracle_cso_generation.argtypes = [i32, i64, i64, i64, u64, u64, f32, P, P, P, P, P, P,
                                            i32]
        L.oracle_de_indices.argtypes = [i64, i64, u64, u64, P]
        L.oracle_de_jrand.argtypes = [i64, i64, u64, u64]
        L.oracle_de_jrand.restype = i64
        L.oracle_de_trial_with.argtypes = [i64, P, P, P, P, P, i64, f32, f32, P, P, P]
        L.oracle_de_generation.argtypes = [i32, i64, i64, P, P, P, f32, f32, u64, u64, P, P, i32]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float32)
    if shape is not None:
        a = a.reshape(shape)
    return a


def _bounds(lb, ub, D):
    lb = np.broadcast_to(np.asarray(lb, np.float32), (D,)).copy()
    ub = np.broadcast_to(np.asarray(ub, np.float32), (D,)).copy()
    return lb, ub


# ----------------------------------------------------------------- primitives
def philox(ctr, key) -> np.ndarray:
    """Philox4x32-10 of one counter (4 x u32) under key (2 x u32)."""
    c = np.asarray(ctr, np.uint32).copy()
    k = np.asarray(key, np.uint32).copy()
    out = np.zeros(4, np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def uniform24(b: int) -> float:
    return float(np.float32(lib().oracle_uniform24(int(b) & 0xFFFFFFFF)))


def draw(rows, D, row0, t, tag, seed) -> np.ndarray:
    R = np.zeros((rows, D), np.float32)
    lib().oracle_draw(rows, D, row0, t, tag, seed, _p(R))
    return R


def evaluate(problem, X, threads: int = 1) -> np.ndarray:
    """fp64 textbook fitness of every row of X (fp32 [rows x D])."""
    problem = PROBLEMS.get(problem, problem)
    X = _f32(X)
    if X.ndim == 1:
        X = X.reshape(1, -1)
    F = np.zeros(X.shape[0], np.float64)
    lib().oracle_eval(int(problem), X.shape[0], X.shape[1], _p(X), _p(F), threads)
    return F


def pso_init(rows, D, row0, lb, ub, seed):
    lb, ub = _bounds(lb, ub, D)
    X = np.zeros((rows, D), np.float32)
    V = np.zeros((rows, D), np.float32)
    lib().oracle_pso_init(rows, D, row0, _p(lb), _p(ub), seed, _p(X), _p(V))
    return X, V


def pso_move_with(X, V, P, G, R1, R2, w, phi_p, phi_g, lb, ub):
    """In-place move with injected r1/r2 (the test hook of the hand-worked example)."""
    rows, D = X.shape
    lb, ub = _bounds(lb, ub, D)
    G = _f32(G)
    R1 = _f32(np.broadcast_to(R1, X.shape))
    R2 = _f32(np.broadcast_to(R2, X.shape))
    lib().oracle_pso_move_with(rows, D, _p(X), _p(V), _p(_f32(P)), _p(G), _p(R1), _p(R2),
                               w, phi_p, phi_g, _p(lb), _p(ub))


def pso_move(X, V, P, G, row0, t, seed, w, phi_p, phi_g, lb, ub, threads=1):
    rows, D = X.shape
    lb, ub = _bounds(lb, ub, D)
    lib().oracle_pso_move(rows, D, row0, t, seed, _p(X), _p(V), _p(_f32(P)), _p(_f32(G)),
                          w, phi_p, phi_g, _p(lb), _p(ub), threads)


def pso_tell_rows(X, f, P, pf):
    rows, D = X.shape
    imp = np.zeros(rows, np.uint8)
    lib().oracle_pso_tell_rows(rows, D, _p(X), _p(_f32(f)), _p(P), _p(pf), _p(imp))
    return imp


def argmin(f) -> tuple[int, float]:
    f = _f32(f)
    m = np.zeros(1, np.float32)
    i = lib().oracle_argmin(f.shape[0], _p(f), _p(m))
    return int(i), float(m[0])


def pso_tell(X, f, P, pf, G, gf, gidx, W=1):
    """Unified tell of one generation (oracle_pso_tell), in place on P, pf, G.
    Returns (gf, gidx, hist_t)."""
    N, D = X.shape
    gfa = np.array([gf], np.float32)
    gia = np.array([gidx], np.int64)
    h = np.zeros(1, np.float32)
    lib().oracle_pso_tell(N, D, W, _p(_f32(X)), _p(_f32(f)), _p(P), _p(pf), _p(G), _p(gfa),
                          _p(gia), _p(h))
    return float(gfa[0]), int(gia[0]), float(h[0])


def pso_run_with(problem, X, V, R1, R2, n_gens, w, phi_p, phi_g, lb, ub, W=1) -> PSOState:
    """The stateful driver from a caller-supplied unevaluated (X, V) with injected r1/r2
    (broadcast to [n_gens x N x D]); returns the state after n_gens generations."""
    problem = PROBLEMS.get(problem, problem)
    X = _f32(X).copy(); V = _f32(V).copy()
    N, D = X.shape
    lb, ub = _bounds(lb, ub, D)
    R1 = _f32(np.broadcast_to(np.asarray(R1, np.float32), (max(n_gens, 1), N, D)))
    R2 = _f32(np.broadcast_to(np.asarray(R2, np.float32), (max(n_gens, 1), N, D)))
    P = np.zeros_like(X); pf = np.zeros(N, np.float32); f = np.zeros(N, np.float32)
    F64 = np.zeros(N); G = np.zeros(D, np.float32)
    gf = np.zeros(1, np.float32); gidx = np.zeros(1, np.int64)
    hist = np.zeros(n_gens + 1, np.float32)
    lib().oracle_pso_run_with(int(problem), N, D, _p(lb), _p(ub), w, phi_p, phi_g, n_gens, W,
                              _p(X), _p(V), _p(P), _p(pf), _p(f), _p(F64), _p(G), _p(gf),
                              _p(gidx), _p(hist), _p(R1), _p(R2))
    return PSOState(int(problem), N, D, lb, ub, w, phi_p, phi_g, 0, X, V, P, pf, f, F64, G,
                    float(gf[0]), int(gidx[0]), n_gens, [float(v) for v in hist])


def cso_perm(x, B, blk, t, seed) -> int:
    return int(lib().oracle_cso_perm(x, B, blk, t, seed))


def cso_pairs(B, blk, t, seed) -> np.ndarray:
    """All pairs (local indices) of one block: [[pi(0), pi(1)], [pi(2), pi(3)], ...]."""
    perm = np.array([cso_perm(x, B, blk, t, seed) for x in range(B)], np.int64)
    return perm[: 2 * (B // 2)].reshape(-1, 2)


# ------------------------------------------------------------ stateful PSO
@dataclass
class PSOState:
    """Dense oracle state at rest after evaluation (R-2)."""
    problem: int
    N: int
    D: int
    lb: np.ndarray
    ub: np.ndarray
    w: float
    phi_p: float
    phi_g: float
    seed: int
    X: np.ndarray
    V: np.ndarray
    P: np.ndarray
    pf: np.ndarray
    f: np.ndarray
    F64: np.ndarray
    G: np.ndarray
    gf: float
    gidx: int
    t: int
    hist: list = field(default_factory=list)

    def copy(self) -> "PSOState":
        return PSOState(self.problem, self.N, self.D, self.lb.copy(), self.ub.copy(), self.w,
                        self.phi_p, self.phi_g, self.seed, self.X.copy(), self.V.copy(),
                        self.P.copy(), self.pf.copy(), self.f.copy(), self.F64.copy(),
                        self.G.copy(), self.gf, self.gidx, self.t, list(self.hist))


def pso_run(problem, N, D, lb, ub, w=0.6, phi_p=2.5, phi_g=0.8, seed=0, n_gens=0, W=1,
            state: PSOState | None = None, threads=1) -> PSOState:
    """Fresh run (state None): init, evaluate+tell X0, then n_gens x (move, eval, tell).
    With ``state``: continue n_gens generations from it (returns a new state)."""
    problem = PROBLEMS.get(problem, problem)
    lb, ub = _bounds(lb, ub, D)
    L = lib()
    hist = np.zeros(n_gens + 1, np.float32)
    gf = np.zeros(1, np.float32)
    gidx = np.zeros(1, np.int64)
    if state is None:
        X = np.zeros((N, D), np.float32); V = np.zeros_like(X); P = np.zeros_like(X)
        pf = np.zeros(N, np.float32); f = np.zeros(N, np.float32); F64 = np.zeros(N)
        G = np.zeros(D, np.float32)
        fresh, t0, prev_hist = 1, 0, []
    else:
        s = state.copy()
        X, V, P, pf, f, F64, G = s.X, s.V, s.P, s.pf, s.f, s.F64, s.G
        gf[0], gidx[0] = s.gf, s.gidx
        fresh, t0, prev_hist = 0, s.t, s.hist
    L.oracle_pso_run(int(problem), N, D, _p(lb), _p(ub), w, phi_p, phi_g, seed, n_gens, W,
                     fresh, t0, _p(X), _p(V), _p(P), _p(pf), _p(f), _p(F64), _p(G), _p(gf),
                     _p(gidx), _p(hist), threads)
    nh = n_gens + 1 if fresh else n_gens
    return PSOState(int(problem), N, D, lb, ub, w, phi_p, phi_g, seed, X, V, P, pf, f, F64, G,
                    float(gf[0]), int(gidx[0]), t0 + n_gens, prev_hist + [float(h) for h in
                                                                          hist[:nh]])


# ------------------------------------------------------------ stateful CSO
def cso_init(problem, N, D, lb, ub, seed, threads=1):
    """CSO init (R-8): X0 as PSO init, V0 = 0, evaluate all rows."""
    X, V = pso_init(N, D, 0, lb, ub, seed)
    F64 = evaluate(problem, X, threads)
    return X, V, F64.astype(np.float32), F64


def cso_loser_update_with(xw, xl, vl, R1, R2, R3=None, phi=0.0, xbar=None, lb=-np.inf,
                          ub=np.inf):
    """In-place loser update with injected R1/R2/R3 (hand-worked example hook)."""
    D = xl.shape[0]
    lb, ub = _bounds(lb, ub, D)
    R1 = _f32(np.broadcast_to(R1, (D,))); R2 = _f32(np.broadcast_to(R2, (D,)))
    R3 = _f32(np.broadcast_to(0.0 if R3 is None else R3, (D,)))
    xbar = _f32(np.zeros(D) if xbar is None else xbar)
    lib().oracle_cso_loser_update_with(D, _p(_f32(xw)), _p(xl), _p(vl), _p(R1), _p(R2), _p(R3),
                                       phi, _p(xbar), _p(lb), _p(ub))


def cso_generation(problem, X, V, f, F64, B, t, seed, lb, ub, phi=0.0, threads=1):
    """One CSO generation at t, in place."""
    problem = PROBLEMS.get(problem, problem)
    N, D = X.shape
    lb, ub = _bounds(lb, ub, D)
    lib().oracle_cso_generation(int(problem), N, D, B, t, seed, phi, _p(lb), _p(ub), _p(X),
                                _p(V), _p(f), _p(F64), threads)


# --------------------------------------------------------------------- DE
def de_indices(N, i, t, seed) -> list:
    out = np.zeros(3, np.int64)
    lib().oracle_de_indices(N, i, t, seed, _p(out))
    return [int(v) for v in out]


def de_jrand(D, i, t, seed) -> int:
    return int(lib().oracle_de_jrand(D, i, t, seed))


def de_trial_with(xi, xa, xb, xc, U, jrand, F, CR, lb=-np.inf, ub=np.inf):
    """DE/rand/1/bin trial with injected crossover uniforms (hand-worked example hook)."""
    D = len(xi)
    lb, ub = _bounds(lb, ub, D)
    u = np.zeros(D, np.float32)
    lib().oracle_de_trial_with(D, _p(_f32(xi)), _p(_f32(xa)), _p(_f32(xb)), _p(_f32(xc)),
                               _p(_f32(np.broadcast_to(U, (D,)))), jrand, F, CR, _p(lb), _p(ub),
                               _p(u))
    return u


def de_init(problem, N, D, lb, ub, seed, threads=1):
    """DE init (R-14): X0 as PSO init (tag 0), evaluate all rows."""
    X, _ = pso_init(N, D, 0, lb, ub, seed)
    F64 = evaluate(problem, X, threads)
    return X, F64.astype(np.float32), F64


def de_generation(problem, X, f, F64, t, seed, lb, ub, F=0.5, CR=0.9, threads=1):
    """One synchronous DE generation at t, in place."""
    problem = PROBLEMS.get(problem, problem)
    N, D = X.shape
    lb, ub = _bounds(lb, ub, D)
    lib().oracle_de_generation(int(problem), N, D, _p(X), _p(f), _p(F64), F, CR, t, seed, _p(lb),
                               _p(ub), threads)
