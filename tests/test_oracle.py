"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names the passage / reading it pins.  A plausible mistake in the
oracle (dropped term, wrong sign, off-by-one index, transposed operand,
wrong tie rule, wrong counter layout) fails at least one of these.
"""
import math
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.filterwarnings("ignore")


# ---------------------------------------------------------------- Philox
def _kat(golden_dir):
    rows = []
    for line in open(os.path.join(golden_dir, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


def test_philox_known_answers(golden_dir):
    """Random123 kat_vectors (SURVEY §8(c) Philox pin)."""
    kat = _kat(golden_dir)
    assert len(kat) == 3
    for ctr, key, out in kat:
        assert list(O.philox(ctr, key)) == out


def test_uniform24_edges():
    """R-6: top 24 bits scaled by 2^-24, range [0,1)."""
    assert O.uniform24(0) == 0.0
    assert O.uniform24(0xFF) == 0.0  # low 8 bits discarded
    assert O.uniform24(0x80000000) == 0.5
    assert O.uniform24(0x100) == 2.0 ** -24
    assert O.uniform24(0xFFFFFFFF) == 1.0 - 2.0 ** -24


def test_draw_counter_layout():
    """R-6: R[r][j] uses ctr = (j//4, row0+r, t, tag) and word j%4 (KAT-pinned Philox)."""
    seed = (0x1234567 << 32) | 0x89ABCDEF
    R = O.draw(3, 9, 5, 7, 3, seed)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for r in range(3):
        for j in range(9):
            w = O.philox([j // 4, 5 + r, 7, 3], key)[j % 4]
            assert R[r, j] == np.float32((int(w) >> 8) * 2.0 ** -24)
    # different tag / generation / row offset give different streams
    assert not np.array_equal(R, O.draw(3, 9, 5, 7, 2, seed))
    assert not np.array_equal(R, O.draw(3, 9, 5, 8, 3, seed))
    assert not np.array_equal(R, O.draw(3, 9, 6, 7, 3, seed))


def test_uniform_statistics():
    """S:128-134 mean 0.5 +- 0.005 over 1e6 draws; S:92 chi^2 over 100 bins, p > 0.001."""
    R = O.draw(1000, 1000, 0, 0, 2, 0).ravel().astype(np.float64)
    assert R.min() >= 0.0 and R.max() < 1.0
    assert abs(R.mean() - 0.5) < 0.005
    counts = np.histogram(R, bins=100, range=(0.0, 1.0))[0]
    chi2 = float(((counts - 1e4) ** 2 / 1e4).sum())
    # chi^2_{99} upper 0.001 quantile = 148.23
    assert chi2 < 148.23


# ------------------------------------------------------------- functions
def _ev(name, x):
    return float(O.evaluate(name, np.asarray(x, np.float32).reshape(1, -1))[0])


def test_sphere_closed_form():
    """Sphere(0) = 0; Sphere(1,2,3) = 14."""
    assert _ev("sphere", [0.0] * 7) == 0.0
    assert _ev("sphere", [1, 2, 3]) == 14.0
    assert _ev("sphere", [-3, 4]) == 25.0


def test_ackley_closed_forms():
    """Ackley(0)=0; at integer vectors cos(2 pi k)=1 so f = 20(1-exp(-0.2 sqrt(sum k^2/D)));
    at x = 1/2 * ones, cos(pi) = -1 so f = 20 + e - 20 exp(-0.1) - exp(-1)."""
    assert abs(_ev("ackley", [0.0] * 10)) < 1e-12
    for k in (1, 2, -3):
        assert abs(_ev("ackley", [k] * 5) - 20 * (1 - math.exp(-0.2 * abs(k)))) < 1e-12
    k = [1, -2, 3, 0]
    ref = 20 * (1 - math.exp(-0.2 * math.sqrt(sum(v * v for v in k) / 4)))
    assert abs(_ev("ackley", k) - ref) < 1e-12
    assert abs(_ev("ackley", [1.0] * 5) - 3.6253849384403627) < 1e-12
    ref = 20 + math.e - 20 * math.exp(-0.1) - math.exp(-1)
    assert abs(_ev("ackley", [0.5] * 6) - ref) < 1e-12


def test_rastrigin_closed_forms():
    """Integer lattice: f(k) = sum k^2 exactly-ish; x = 1/2: 10 + 1/4 + 10 per dim."""
    assert abs(_ev("rastrigin", [0.0] * 9)) < 1e-12
    k = [3, -4, 5, 1, 0, -7]
    assert abs(_ev("rastrigin", k) - sum(v * v for v in k)) < 1e-9
    assert abs(_ev("rastrigin", [0.5, -0.5]) - 2 * 20.25) < 1e-12


def test_griewank_closed_forms():
    """f(0)=0; 1-based index: x=(0, pi*sqrt2) -> 1 + 2pi^2/4000 - (1*cos(pi)) = 2 + pi^2/2000."""
    assert abs(_ev("griewank", [0.0] * 12)) < 1e-15
    x1 = np.float32(math.pi * math.sqrt(2.0))
    ref = 1 + float(x1) ** 2 / 4000 - math.cos(float(x1) / math.sqrt(2.0))
    assert abs(_ev("griewank", [0.0, x1]) - ref) < 1e-12
    assert abs(_ev("griewank", [0.0, x1]) - (2 + math.pi ** 2 / 2000)) < 1e-6
    # x_j = 2 pi m_j sqrt(j+1): every cosine = 1 -> f ~= sum x^2 / 4000
    m = [1, -2, 1, 3]
    x = [np.float32(2 * math.pi * mj * math.sqrt(j + 1)) for j, mj in enumerate(m)]
    assert abs(_ev("griewank", x) - sum(float(v) ** 2 for v in x) / 4000) < 1e-9


def test_rosenbrock_closed_forms():
    """f(1)=0; f(0)=D-1; D=1 -> 0; f(a, a^2) = (1-a)^2; f(-1, 1) = 4."""
    assert _ev("rosenbrock", [1.0] * 8) == 0.0
    assert _ev("rosenbrock", [0.0] * 8) == 7.0
    assert _ev("rosenbrock", [3.5]) == 0.0
    assert _ev("rosenbrock", [-1.0, 1.0]) == 4.0
    assert _ev("rosenbrock", [2.0, 4.0]) == 1.0
    # x_{j+1} - x_j^2 (not x_j - x_{j+1}^2): (0, 1) -> 100 + 1
    assert _ev("rosenbrock", [0.0, 1.0]) == 101.0


def test_row_permutation_equivariance():
    """row i of the fitness depends only on row i."""
    rng = np.random.default_rng(3)
    X = rng.uniform(-5, 5, (37, 13)).astype(np.float32)
    perm = rng.permutation(37)
    for p in O.PROBLEMS:
        F = O.evaluate(p, X)
        assert np.array_equal(O.evaluate(p, X[perm]), F[perm])


def test_eval_threads_invariant():
    rng = np.random.default_rng(4)
    X = rng.uniform(-5, 5, (64, 33)).astype(np.float32)
    for p in O.PROBLEMS:
        assert np.array_equal(O.evaluate(p, X, threads=1), O.evaluate(p, X, threads=4))


# ------------------------------------------------------------------- PSO
def _golden_pso(golden_dir):
    g = {}
    for line in open(os.path.join(golden_dir, "pso_two_particle.txt")):
        if line.startswith("#") or not line.strip():
            continue
        tok = line.split()
        if tok[0] in ("X0", "V0"):
            g[tok[0]] = np.array([float(v) for v in tok[1:]], np.float32).reshape(2, 2)
        elif tok[0] == "gen":
            t = int(tok[1])
            f = [float(tok[3]), float(tok[4])]
            gb = int(tok[6])
            X = np.array([float(v) for v in tok[8:12]], np.float32).reshape(2, 2)
            V = np.array([float(v) for v in tok[13:17]], np.float32).reshape(2, 2)
            g[t] = (f, gb, X, V)
    return g


def test_pso_hand_worked_two_particles(golden_dir):
    """SURVEY §8(c) dyadic example: three generations of evaluate -> tell -> move."""
    g = _golden_pso(golden_dir)
    X, V = g["X0"].copy(), g["V0"].copy()
    P = X.copy()
    pf = np.full(2, np.inf, np.float32)
    G = np.zeros(2, np.float32)
    gf, gidx = np.inf, -1
    for t in range(3):
        F = O.evaluate("sphere", X)
        f = F.astype(np.float32)
        assert list(F) == g[t][0]
        O.pso_tell_rows(X, f, P, pf)
        i, fm = O.argmin(f)
        if fm < gf:
            gf, gidx, G = fm, i, X[i].copy()
        assert gidx == g[t][1]
        O.pso_move_with(X, V, P, G, 0.5, 0.25, 0.5, 2.0, 1.0, -4.0, 4.0)
        assert np.array_equal(X, g[t][2]), (t, X)
        assert np.array_equal(V, g[t][3]), (t, V)
    # gbest after gen 2 is particle 0's X2 = (3/16, 27/32)
    assert np.array_equal(G, np.array([0.1875, 0.84375], np.float32))
    assert gf == np.float32(765 / 1024)
    # pbest: particle 0 improved every generation; particle 1 kept X0
    assert np.array_equal(P[1], [-1.0, 0.5])
    assert pf[1] == 1.25


def test_pso_hand_worked_through_driver(golden_dir):
    """The same golden trajectory replayed through the oracle's stateful C driver
    (oracle_pso_run_with: the driver oracle_pso_run uses, with r1/r2 injected).  Pins the
    driver's generation order evaluate -> tell (pbest, then gbest) -> move of Listing 1
    P:243-277 / Eqs. (1)-(3) P:443-447 (R-2): any other order changes gen 1's fitness."""
    g = _golden_pso(golden_dir)
    for n in range(4):
        s = O.pso_run_with("sphere", g["X0"], g["V0"], 0.5, 0.25, n, 0.5, 2.0, 1.0, -4.0, 4.0)
        # hist[t] = min f32 of generation t (gens 0..n evaluated; golden f up to gen 2)
        k = min(n + 1, 3)
        assert len(s.hist) == n + 1
        assert s.hist[:k] == [min(g[t][0]) for t in range(k)]
        if n == 0:
            assert np.array_equal(s.X, g["X0"]) and np.array_equal(s.V, g["V0"])
            assert list(s.f) == g[0][0] and s.gidx == g[0][1]
        else:
            assert np.array_equal(s.X, g[n - 1][2]), (n, s.X)
            assert np.array_equal(s.V, g[n - 1][3]), (n, s.V)
            if n < 3:
                assert list(s.f) == g[n][0] and s.gidx == g[n][1]
    s = O.pso_run_with("sphere", g["X0"], g["V0"], 0.5, 0.25, 2, 0.5, 2.0, 1.0, -4.0, 4.0)
    # after generation 2's tell: gbest = particle 0's X2 = (3/16, 27/32), f = 765/1024
    assert s.gidx == 0 and s.gf == np.float32(765 / 1024)
    assert np.array_equal(s.G, np.array([0.1875, 0.84375], np.float32))
    assert np.array_equal(s.P[1], [-1.0, 0.5]) and s.pf[1] == 1.25
    assert np.array_equal(s.P[0], s.G)


def test_pso_tell_gbest_strict_against_incumbent():
    """S:316 "strict improvement; ties keep incumbent" for gbest (SURVEY §8(c) argmin pin):
    a generation whose minimum EQUALS the incumbent gf must not move G or gidx."""
    X = np.array([[1.0, 1.0], [2.0, 2.0], [3.0, 3.0]], np.float32)
    G = np.array([9.0, 9.0], np.float32)
    P = X.copy(); pf = np.full(3, np.inf, np.float32)
    gf, gidx, h = O.pso_tell(X, np.array([4.0, 2.0, 2.0], np.float32), P, pf, G, 2.0, 7)
    assert (gf, gidx, h) == (2.0, 7, 2.0)
    assert np.array_equal(G, [9.0, 9.0])
    # a strictly better minimum moves it, to the lowest index among the tying rows
    gf, gidx, h = O.pso_tell(X, np.array([4.0, 1.5, 1.5], np.float32), P, pf, G, 2.0, 7)
    assert (gf, gidx, h) == (1.5, 1, 1.5)
    assert np.array_equal(G, X[1])
    # NaN ranks as +inf: an all-NaN generation never moves gbest, hist = +inf
    gf, gidx, h = O.pso_tell(X, np.full(3, np.nan, np.float32), P, pf, G, 1.5, 1)
    assert (gf, gidx) == (1.5, 1) and h == np.inf


@pytest.mark.parametrize("W", [2, 3, 4])
def test_pso_tell_shard_combine_ties_lowest_global_index(W):
    """S:349 / S:285 / R-11: equal shard winners are combined to the LOWEST global index
    (the first shard), whatever W; within a shard the lowest index wins too."""
    N, D = 12, 3
    X = np.arange(N * D, dtype=np.float32).reshape(N, D)
    f = np.full(N, 5.0, np.float32)
    bounds = np.cumsum([0] + [N // W + (s < N % W) for s in range(W)])
    # plant the same minimum as the LAST row of every shard
    for s in range(W):
        f[bounds[s + 1] - 1] = 1.0
    P = X.copy(); pf = np.full(N, np.inf, np.float32); G = np.zeros(D, np.float32)
    gf, gidx, h = O.pso_tell(X, f, P, pf, G, np.inf, -1, W=W)
    assert gidx == bounds[1] - 1 and gf == 1.0 and np.array_equal(G, X[gidx])
    # and the same answer as W = 1 (sharding invariance)
    P = X.copy(); pf = np.full(N, np.inf, np.float32); G1 = np.zeros(D, np.float32)
    assert O.pso_tell(X, f, P, pf, G1, np.inf, -1, W=1)[1] == gidx


def test_pso_clip_case():
    """R-4: positions clipped, velocity NOT clamped (SURVEY §8(c) clip case)."""
    X = np.array([[1.5]], np.float32); V = np.array([[1.0]], np.float32)
    O.pso_move_with(X, V, X.copy(), X[0].copy(), 0.3, 0.7, 0.5, 2.5, 0.8, -2.0, 1.75)
    assert X[0, 0] == 1.75 and V[0, 0] == 0.5
    X = np.array([[-1.5]], np.float32); V = np.array([[-1.0]], np.float32)
    O.pso_move_with(X, V, X.copy(), X[0].copy(), 0.3, 0.7, 0.5, 2.5, 0.8, -1.75, 2.0)
    assert X[0, 0] == -1.75 and V[0, 0] == -0.5


def test_pso_fixed_point_and_w0():
    """S:319 x = pbest = gbest, v = 0 -> x unchanged; S:320 w=0 at gbest -> v stays 0."""
    rng = np.random.default_rng(0)
    X = rng.uniform(-1, 1, (1, 6)).astype(np.float32)
    X0 = X.copy(); V = np.zeros_like(X)
    R1 = rng.random((1, 6)); R2 = rng.random((1, 6))
    O.pso_move_with(X, V, X0, X0[0], R1, R2, 0.6, 2.5, 0.8, -2, 2)
    assert np.array_equal(X, X0) and not V.any()
    V = rng.uniform(-1, 1, X.shape).astype(np.float32)
    O.pso_move_with(X, V, X0, X0[0], R1, R2, 0.0, 2.5, 0.8, -2, 2)
    assert not V.any() and np.array_equal(X, X0)


def test_pso_move_terms_separately():
    """Each term of v alone (one-hot coefficients) -- catches swapped/sign-flipped terms."""
    X = np.array([[1.0, -2.0]], np.float32)
    P = np.array([[3.0, 0.0]], np.float32)
    G = np.array([-1.0, 4.0], np.float32)
    V0 = np.array([[0.5, 0.25]], np.float32)
    for (w, pp, pg), v_expect in (((1, 0, 0), [0.5, 0.25]), ((0, 1, 0), [2.0, 2.0]),
                                  ((0, 0, 1), [-2.0, 6.0])):
        Xc, Vc = X.copy(), V0.copy()
        O.pso_move_with(Xc, Vc, P, G, 1.0, 1.0, w, pp, pg, -100, 100)
        assert np.array_equal(Vc[0], v_expect)
        assert np.array_equal(Xc[0], X[0] + np.array(v_expect, np.float32))
    # r1 multiplies the pbest term, r2 the gbest term
    Xc, Vc = X.copy(), V0.copy()
    O.pso_move_with(Xc, Vc, P, G, 0.5, 0.0, 0.0, 1.0, 1.0, -100, 100)
    assert np.array_equal(Vc[0], [1.0, 1.0])


def test_pso_tell_strict_and_nan():
    """S:316 strict improvement, ties keep the incumbent; NaN never improves (R-5)."""
    X = np.arange(8, dtype=np.float32).reshape(4, 2)
    P = np.zeros_like(X)
    pf = np.array([1.0, 1.0, 1.0, np.inf], np.float32)
    imp = O.pso_tell_rows(X, np.array([0.5, 1.0, np.nan, np.nan], np.float32), P, pf)
    assert list(imp) == [1, 0, 0, 0]
    assert np.array_equal(P[0], X[0]) and not P[1:].any()
    assert list(pf) == [0.5, 1.0, 1.0, np.inf]


def test_argmin_brute_force_with_ties():
    """lowest index on ties; NaN as +inf; brute force on N <= 64."""
    rng = np.random.default_rng(7)
    for trial in range(200):
        n = int(rng.integers(1, 65))
        f = rng.integers(0, 5, n).astype(np.float32)  # many ties
        if trial % 3 == 0:
            f[rng.integers(0, n)] = np.nan
        if trial % 7 == 0:
            f[:] = np.nan
        i, m = O.argmin(f)
        vals = [np.inf if np.isnan(v) else float(v) for v in f]
        best = min(vals)
        assert m == best
        assert i == vals.index(best)
    assert O.argmin(np.array([-0.0, 0.0], np.float32))[0] == 0
    assert O.argmin(np.array([0.0, -0.0], np.float32))[0] == 0


def test_pso_init_in_bounds_and_seeded():
    lb = np.array([-1, 0, 5, -600], np.float32); ub = np.array([1, 3, 6, 600], np.float32)
    X, V = O.pso_init(500, 4, 0, lb, ub, 11)
    assert (X >= lb).all() and (X <= ub).all() and not V.any()
    X2, _ = O.pso_init(500, 4, 0, lb, ub, 11)
    X3, _ = O.pso_init(500, 4, 0, lb, ub, 12)
    assert np.array_equal(X, X2) and not np.array_equal(X, X3)
    assert np.allclose(X.mean(0), (lb + ub) / 2, atol=0.1 * (ub - lb).max())
    # row offset: rows 100.. of a full init equal an init started at row0=100
    Xs, _ = O.pso_init(50, 4, 100, lb, ub, 11)
    assert np.array_equal(Xs, X[100:150])


@pytest.mark.parametrize("problem,lb,ub", [("sphere", -5.12, 5.12), ("ackley", -32.768, 32.768),
                                           ("rastrigin", -5.12, 5.12),
                                           ("griewank", -600, 600), ("rosenbrock", -5, 10)])
def test_pso_invariants(problem, lb, ub):
    """pf non-increasing; gf non-increasing; gf = min pf; X in bounds."""
    N, D = 40, 9
    s = O.pso_run(problem, N, D, lb, ub, n_gens=0, seed=5)
    prev = s
    for _ in range(15):
        s = O.pso_run(problem, N, D, lb, ub, n_gens=1, seed=5, state=prev)
        assert (s.pf <= prev.pf).all()
        assert s.gf <= prev.gf
        assert s.gf == s.pf.min()
        assert (s.X >= np.float32(lb)).all() and (s.X <= np.float32(ub)).all()
        assert np.array_equal(s.P[s.gidx], s.G)
        assert s.hist[-1] == s.f.min()
        prev = s


def test_pso_split_equals_single_run():
    """step(a) then step(b) == step(a+b) bitwise (S:531 purity)."""
    a = O.pso_run("ackley", 30, 7, -32.768, 32.768, n_gens=12, seed=3)
    b = O.pso_run("ackley", 30, 7, -32.768, 32.768, n_gens=5, seed=3)
    b = O.pso_run("ackley", 30, 7, -32.768, 32.768, n_gens=7, seed=3, state=b)
    for k in ("X", "V", "P", "pf", "f", "G"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.hist == b.hist and a.gf == b.gf and a.gidx == b.gidx


@pytest.mark.parametrize("W", [2, 3, 4, 8])
def test_pso_simulated_sharding_invariance(W):
    """R-11 / S:574: W contiguous shards give the same trajectory bitwise."""
    a = O.pso_run("rastrigin", 37, 6, -5.12, 5.12, n_gens=20, seed=9, W=1)
    b = O.pso_run("rastrigin", 37, 6, -5.12, 5.12, n_gens=20, seed=9, W=W)
    for k in ("X", "V", "P", "pf", "G"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.hist == b.hist and a.gidx == b.gidx


def test_pso_threads_invariant():
    a = O.pso_run("griewank", 64, 10, -600, 600, n_gens=10, seed=1, threads=1)
    b = O.pso_run("griewank", 64, 10, -600, 600, n_gens=10, seed=1, threads=4)
    assert np.array_equal(a.X, b.X) and a.hist == b.hist


def test_pso_convergence_smoke():
    """10-D Sphere, pop 100, 500 iterations -> best < 1e-4 (convergence, not parity)."""
    s = O.pso_run("sphere", 100, 10, -5.12, 5.12, n_gens=500, seed=0)
    assert s.gf < 1e-4
    assert s.hist[0] > 1.0


# ------------------------------------------------------------------- CSO
@pytest.mark.parametrize("B", [2, 3, 5, 16, 100, 625, 4096, 6250])
def test_cso_perm_is_bijection(B):
    """R-8: the keyed Feistel + cycle-walking map is a permutation of [0,B)."""
    for blk, t in ((0, 0), (3, 17)):
        perm = sorted(O.cso_perm(x, B, blk, t, 42) for x in range(B))
        assert perm == list(range(B))


def test_cso_perm_exhaustive_65536():
    perm = np.array([O.cso_perm(x, 65536, 1, 2, 7) for x in range(65536)])
    assert np.array_equal(np.sort(perm), np.arange(65536))
    # keyed: another generation gives another matching
    perm2 = np.array([O.cso_perm(x, 65536, 1, 3, 7) for x in range(64)])
    assert not np.array_equal(perm[:64], perm2)


def test_cso_hand_worked_pair(golden_dir):
    g = {}
    for line in open(os.path.join(golden_dir, "cso_one_pair.txt")):
        if line.startswith("#") or not line.strip():
            continue
        tok = line.split()
        g[tok[0]] = np.array([float(v) for v in tok[1:]], np.float32)
    xl, vl = g["xl"].copy(), g["vl"].copy()
    O.cso_loser_update_with(g["xw"], xl, vl, g["R1"][0], g["R2"][0])
    assert np.array_equal(vl, g["v_new"]) and np.array_equal(xl, g["x_new"])
    assert _ev("sphere", xl) == g["sphere"][0]
    # the mean-position term (phi != 0): xbar = xl -> term vanishes; xbar = xl + 1 -> + phi*R3
    xl2, vl2 = g["xl"].copy(), g["vl"].copy()
    O.cso_loser_update_with(g["xw"], xl2, vl2, 0.5, 0.25, R3=0.5, phi=0.5, xbar=g["xl"] + 1)
    assert np.array_equal(vl2, g["v_new"] + np.float32(0.25))


@pytest.mark.parametrize("N,B", [(64, 8), (64, 64), (50, 16), (33, 33)])
def test_cso_generation_invariants(N, B):
    """Winners bitwise unchanged; floor(Bb/2) losers per block; min f non-increasing;
    the loser is the worse of its pair (ties -> lower index wins); X in bounds."""
    D, seed = 7, 13
    X, V, f, F64 = O.cso_init("rastrigin", N, D, -5.12, 5.12, seed)
    for t in range(6):
        X0, V0, f0 = X.copy(), V.copy(), f.copy()
        O.cso_generation("rastrigin", X, V, f, F64, B, t, seed, -5.12, 5.12)
        changed = set(np.nonzero((X != X0).any(1) | (V != V0).any(1))[0].tolist())
        losers = set()
        for blk in range((N + B - 1) // B):
            Bb = min(B, N - blk * B)
            for a, b in O.cso_pairs(Bb, blk, t, seed):
                i, k = blk * B + a, blk * B + b
                lo = k if (f0[i] < f0[k] or (f0[i] == f0[k] and i < k)) else i
                losers.add(int(lo))
        assert changed <= losers
        assert len(losers) == sum(min(B, N - b * B) // 2 for b in range((N + B - 1) // B))
        assert f.min() <= f0.min()
        assert (X >= np.float32(-5.12)).all() and (X <= np.float32(5.12)).all()
        assert np.array_equal(f, O.evaluate("rastrigin", X).astype(np.float32))


def test_cso_tie_goes_to_lower_global_index():
    """R-8: equal fitness -> the LOWER global index wins and passes unchanged.  Every row
    is a sign pattern of one vector a (Sphere f = sum a^2 for all rows, exactly), so every
    pair is a tie: the higher index of each pair must be the (only) one that moves."""
    rng = np.random.default_rng(21)
    N, D, B, seed = 64, 9, 16, 5
    a = rng.uniform(0.5, 2.0, D).astype(np.float32)
    X = (a * rng.choice([-1.0, 1.0], (N, D))).astype(np.float32)
    V = np.zeros_like(X)
    F64 = O.evaluate("sphere", X); f = F64.astype(np.float32)
    assert (f == f[0]).all()
    X0 = X.copy()
    O.cso_generation("sphere", X, V, f, F64, B, 3, seed, -5.12, 5.12)
    for blk in range(N // B):
        for p, q in O.cso_pairs(B, blk, 3, seed):
            lo, hi = blk * B + min(p, q), blk * B + max(p, q)
            assert np.array_equal(X[lo], X0[lo]), (lo, hi)
            if not np.array_equal(X0[lo], X0[hi]):
                assert not np.array_equal(X[hi], X0[hi]), (lo, hi)


@pytest.mark.parametrize("B", [8, 32])
def test_cso_xbar_is_the_column_mean(B):
    """[CSO] Eq. (6) (R-8, R-15): xbar is the population MEAN position.  Closed forms:
    (1) all rows equal -> xbar = that row, every difference is 0 and V0 = 0, so nothing
    moves for any phi; (2) rows +-x in equal numbers -> xbar = 0 exactly, so each loser
    follows the update with xbar = 0."""
    N, D, seed = 32, 5, 3
    row = np.array([1.5, -2.0, 0.25, 3.0, -0.5], np.float32)
    X = np.tile(row, (N, 1)); V = np.zeros_like(X)
    F64 = O.evaluate("sphere", X); f = F64.astype(np.float32)
    O.cso_generation("sphere", X, V, f, F64, B, 0, seed, -5.12, 5.12, phi=0.3)
    assert np.array_equal(X, np.tile(row, (N, 1))) and not V.any()
    # (2) half +x, half -x: column mean 0
    rng = np.random.default_rng(2)
    H = rng.uniform(-4, 4, (N // 2, D)).astype(np.float32)
    X = np.concatenate([H, -H]); X = X[rng.permutation(N)]
    V = rng.uniform(-1, 1, (N, D)).astype(np.float32)
    F64 = O.evaluate("sphere", X); f = F64.astype(np.float32)
    X0, V0, f0 = X.copy(), V.copy(), f.copy()
    t, phi = 4, 0.3
    O.cso_generation("sphere", X, V, f, F64, B, t, seed, -5.12, 5.12, phi=phi)
    for blk in range(N // B):
        for p, q in O.cso_pairs(B, blk, t, seed):
            i, k = blk * B + p, blk * B + q
            w, l = (i, k) if (f0[i] < f0[k] or (f0[i] == f0[k] and i < k)) else (k, i)
            R = [O.draw(1, D, l, t, tag, seed)[0] for tag in (5, 6, 7)]
            xl, vl = X0[l].copy(), V0[l].copy()
            O.cso_loser_update_with(X0[w], xl, vl, R[0], R[1], R[2], phi=phi,
                                    xbar=np.zeros(D, np.float32), lb=-5.12, ub=5.12)
            assert np.array_equal(X[l], xl) and np.array_equal(V[l], vl), (l, w)
            assert np.array_equal(X[w], X0[w])


# -------------------------------------------------------------------- DE
def test_de_spec_examples(golden_dir):
    """S:328-329 (golden/de_examples.txt): mutant = x_a + F (x_b - x_c)."""
    for line in open(os.path.join(golden_dir, "de_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [float(x) for x in line.split()]
        F, xa, xb, xc, m = v[0], v[1:3], v[3:5], v[5:7], v[7:9]
        u = O.de_trial_with(np.zeros(2), xa, xb, xc, np.zeros(2), 0, F, 1.0)
        assert list(u) == m


def test_de_crossover_extremes_and_clip():
    xi = np.array([1, 2, 3, 4, 5], np.float32)
    xa = np.array([10, 20, 30, 40, 50], np.float32)
    z = np.zeros(5, np.float32)
    U = np.array([0.1, 0.95, 0.5, 0.99, 0.0], np.float32)
    # CR = 0: only the forced dimension takes the mutant
    assert list(O.de_trial_with(xi, xa, z, z, U, 3, 0.5, 0.0)) == [1, 2, 3, 40, 5]
    # CR = 1: the mutant everywhere
    assert list(O.de_trial_with(xi, xa, z, z, U, 3, 0.5, 1.0)) == [10, 20, 30, 40, 50]
    # U_j < CR picks the mutant (strict), plus j_rand
    assert list(O.de_trial_with(xi, xa, z, z, U, 1, 0.5, 0.5)) == [10, 20, 3, 4, 50]
    # clip to the bounds
    assert list(O.de_trial_with(xi, xa, z, z, U, 1, 0.5, 1.0, lb=0, ub=25)) == [10, 20, 25, 25, 25]
    # F multiplies (x_b - x_c), not (x_c - x_b)
    u = O.de_trial_with(z, z, np.full(5, 3, np.float32), np.full(5, 1, np.float32), U, 0, 0.5, 1.0)
    assert (u == 1.0).all()


def test_de_indices_forced_set_and_distinct():
    """pool 4, exclude 0 -> a permutation of {1,2,3}; no duplicates."""
    for t in range(50):
        for i in range(4):
            r = O.de_indices(4, i, t, 7)
            assert sorted(r) == sorted({0, 1, 2, 3} - {i})
    rng = np.random.default_rng(0)
    for _ in range(2000):
        N = int(rng.integers(4, 10 ** 6))
        i = int(rng.integers(0, N))
        r = O.de_indices(N, i, int(rng.integers(0, 1000)), 3)
        assert len(set(r)) == 3 and i not in r and all(0 <= v < N for v in r)


def test_de_indices_uniform_and_keyed():
    N = 20
    counts = np.zeros(N)
    for t in range(3000):
        for v in O.de_indices(N, 5, t, 11):
            counts[v] += 1
    assert counts[5] == 0
    exp = counts.sum() / (N - 1)
    chi2 = (((counts - exp) ** 2) / exp)[np.arange(N) != 5].sum()
    assert chi2 < 43.8  # chi^2_18, p = 0.001
    assert O.de_indices(1000, 1, 0, 1) != O.de_indices(1000, 1, 1, 1)
    assert O.de_indices(1000, 1, 0, 1) == O.de_indices(1000, 1, 0, 1)
    js = [O.de_jrand(10, i, 0, 2) for i in range(2000)]
    assert min(js) == 0 and max(js) == 9


def test_de_generation_greedy_ties_and_monotone():
    """S:325 trial replaces target iff f(trial) <= f(target); S:330 monotone best."""
    N, D = 30, 6
    X, f, F64 = O.de_init("sphere", N, D, -5.12, 5.12, 9)
    best = [f.min()]
    for t in range(40):
        X0, f0 = X.copy(), f.copy()
        O.de_generation("sphere", X, f, F64, t, 9, -5.12, 5.12)
        changed = (X != X0).any(1)
        assert (f[changed] <= f0[changed]).all() and (f <= f0).all()
        assert np.array_equal(f, O.evaluate("sphere", X).astype(np.float32))
        assert (X >= np.float32(-5.12)).all() and (X <= np.float32(5.12)).all()
        best.append(f.min())
    assert (np.diff(best) <= 0).all() and best[-1] < best[0] * 1e-2
    # ties ("<="): 1-D Sphere on points +-1 with F = 1, CR = 1 and bounds [-1, 1]:
    # every trial clip(x_a + x_b - x_c) is +-1, so f(trial) == f(target) == 1 and EVERY
    # target must be replaced by its trial (a strict "<" would leave X unchanged).
    Xc = np.array([[1.0], [-1.0], [1.0], [1.0], [-1.0], [-1.0], [1.0], [-1.0]], np.float32)
    fc = O.evaluate("sphere", Xc).astype(np.float32)
    Fc = fc.astype(np.float64)
    X0 = Xc.copy()
    O.de_generation("sphere", Xc, fc, Fc, 0, 1, -1, 1, F=1.0, CR=1.0)
    trials = []
    for i in range(8):
        a, b, c = O.de_indices(8, i, 0, 1)
        trials.append(O.de_trial_with(X0[i], X0[a], X0[b], X0[c], [0.5], 0, 1.0, 1.0, -1, 1))
    trials = np.array(trials, np.float32)
    assert np.array_equal(Xc, trials) and not np.array_equal(trials, X0)


def test_de_convergence_smoke():
    X, f, F64 = O.de_init("sphere", 50, 10, -5.12, 5.12, 0)
    for t in range(300):
        O.de_generation("sphere", X, f, F64, t, 0, -5.12, 5.12)
    assert f.min() < 1e-8
