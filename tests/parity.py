"""Parity helpers: GPU state <-> oracle state, tolerances (R-9)."""
from __future__ import annotations

import numpy as np

import oracle as O

RTOL_F, ATOL_F = 1e-5, 1e-6   # fitness: |f - F64| <= max(1e-5 |F64|, 1e-6)
RTOL_X = 1e-6                 # positions: |x - x_or| <= 1e-6 max(|x_or|, 1)


def fit_tol(F64):
    return np.maximum(RTOL_F * np.abs(F64), ATOL_F)


def assert_fitness(f_gpu, F64, what=""):
    f_gpu = np.asarray(f_gpu, np.float64)
    bad = np.abs(f_gpu - F64) > fit_tol(F64)
    # NaN / inf agree by identity
    both_inf = np.isinf(f_gpu) & np.isinf(F64) & (np.sign(f_gpu) == np.sign(F64))
    bad &= ~both_inf
    if bad.any():
        i = int(np.nonzero(bad)[0][0])
        raise AssertionError(f"{what}: {bad.sum()} fitness mismatches, first row {i}: "
                             f"gpu {f_gpu[i]!r} oracle {F64[i]!r}")


def assert_positions(x_gpu, x_or, what=""):
    x_gpu = np.asarray(x_gpu, np.float32)
    diff = np.abs(x_gpu.astype(np.float64) - x_or.astype(np.float64))
    lim = RTOL_X * np.maximum(np.abs(x_or.astype(np.float64)), 1.0)
    bad = diff > lim
    if bad.any():
        idx = tuple(int(v[0]) for v in np.nonzero(bad))
        raise AssertionError(f"{what}: {bad.sum()} position mismatches, first {idx}: "
                             f"gpu {x_gpu[idx]!r} oracle {x_or[idx]!r}")


def gpu_pso_state(pso, D):
    """Dense numpy copy of a PSO handle's (single-shard) state."""
    X = pso.view("X").cpu().numpy()[:, :D].copy()
    V = pso.view("V").cpu().numpy()[:, :D].copy()
    P = pso.view("P").cpu().numpy()[:, :D].copy()
    f = pso.view("F").cpu().numpy().copy()
    pf = pso.view("PF").cpu().numpy().copy()
    G = pso.view("G").cpu().numpy()[:D].copy()
    gf, gidx, _ = pso.best(with_row=False)
    return dict(X=X, V=V, P=P, f=f, pf=pf, G=G, gf=gf, gidx=gidx, hist=pso.history())


def near_tie(a, b):
    """Two fp32 fitness values closer than the tolerance (decision may flip)."""
    a64, b64 = float(a), float(b)
    if not (np.isfinite(a64) and np.isfinite(b64)):
        return False
    return abs(a64 - b64) <= max(RTOL_F * max(abs(a64), abs(b64)), ATOL_F) * 2


def resync_oracle_from_gpu(st: O.PSOState, g: dict) -> O.PSOState:
    """Near-tie protocol (R-9): adopt the GPU's decisions and continue from its state."""
    s = st.copy()
    s.X, s.V, s.P = g["X"].copy(), g["V"].copy(), g["P"].copy()
    s.pf = g["pf"].copy()
    s.f = g["f"].copy()
    s.F64 = O.evaluate(s.problem, s.X)
    s.G = g["G"].copy()
    s.gf, s.gidx = g["gf"], g["gidx"]
    return s


def compare_pso(g: dict, st: O.PSOState, prev_pf_gpu=None, label=""):
    """Compare a GPU state against the oracle state.  Returns the list of
    near-tie decision flips found (empty if the states agree).  Raises on any
    disagreement that is not explained by a near-tie."""
    flips = []
    assert_positions(g["X"], st.X, f"{label} X")
    assert_positions(g["V"], st.V, f"{label} V")
    # fitness of the GPU's population vs the fp64 textbook value of the same rows
    assert_fitness(g["f"], O.evaluate(st.problem, g["X"]), f"{label} f")
    # pbest decisions: rows whose pbest differs must be near-ties
    pd = np.nonzero((g["P"] != st.P).any(1))[0]
    for i in pd:
        if not near_tie(g["f"][i], st.pf[i] if prev_pf_gpu is None else prev_pf_gpu[i]):
            raise AssertionError(f"{label}: pbest of row {i} differs outside a near-tie")
        flips.append(("pbest", int(i)))
    if not pd.size:
        assert_fitness(g["pf"], st.pf.astype(np.float64), f"{label} pf")
    if g["gidx"] != st.gidx:
        if not near_tie(g["gf"], st.gf):
            raise AssertionError(f"{label}: gbest index gpu {g['gidx']} oracle {st.gidx} "
                                 f"(f {g['gf']} vs {st.gf})")
        flips.append(("gbest", g["gidx"], st.gidx))
    else:
        assert np.array_equal(g["G"], st.G), f"{label}: gbest row differs"
    h_or = np.asarray(st.hist, np.float64)
    assert len(g["hist"]) == len(h_or), (len(g["hist"]), len(h_or))
    assert_fitness(g["hist"], h_or, f"{label} hist")
    return flips
