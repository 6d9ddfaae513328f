"""GPU parity of DE/rand/1/bin (R-14) against the CPU oracle."""
import numpy as np
import pytest

import oracle as O
from parity import assert_fitness, near_tie

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2301_12457_b200 as ev  # noqa: E402
from paper_2301_12457_b200 import evox as E  # noqa: E402
from paper_2301_12457_b200 import workloads as WL  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


def _state(de, D):
    return de.view("X").cpu().numpy()[:, :D].copy(), de.view("F").cpu().numpy().copy()


def _de_parity(problem, N, D, seed, gens, F=0.5, CR=0.9, lb=None, ub=None):
    lo, hi = WL.BOUNDS[problem]
    lb = lo if lb is None else lb
    ub = hi if ub is None else ub
    de = ev.DE(N, D, lb, ub, F=F, CR=CR, seed=seed)
    de.step(problem, 0)
    X, f, F64 = O.de_init(problem, N, D, lb, ub, seed)
    Xg, fg = _state(de, D)
    assert np.array_equal(Xg, X)
    assert_fitness(fg, F64, "t=0 f")
    f = fg.copy()  # decisions from here on use the GPU's fp32 fitness
    resync = 0
    for t in range(gens):
        X0 = X.copy()
        de.step(problem, 1)
        O.de_generation(problem, X, f, F64, t, seed, lb, ub, F=F, CR=CR)
        Xg, fg = _state(de, D)
        diff = np.nonzero((Xg != X).any(1))[0]
        for i in diff:
            # a flipped accept/reject decision: both candidates must be near-tied
            r = O.de_indices(N, i, t, seed)
            U = O.draw(1, D, i, t, 10, seed)[0]
            u = O.de_trial_with(X0[i], X0[r[0]], X0[r[1]], X0[r[2]], U, O.de_jrand(D, i, t, seed),
                                F, CR, lb, ub)
            fu = float(O.evaluate(problem, u[None])[0])
            fx = float(O.evaluate(problem, X0[i][None])[0])
            assert near_tie(fu, fx), (t, i, fu, fx)
        if diff.size:
            resync += 1
            X = Xg.copy()
        assert_fitness(fg, O.evaluate(problem, Xg), f"t={t + 1} f")
        f = fg.copy()
        F64 = O.evaluate(problem, X)
    h = de.history()
    assert len(h) == gens + 1 and (np.diff(h) <= 0).all()
    return de, resync


@pytest.mark.parametrize("problem,N,D", [("sphere", 50, 10), ("ackley", 64, 37),
                                         ("rastrigin", 40, 100), ("griewank", 33, 1000),
                                         ("rosenbrock", 20, 4099), ("ackley", 9, 40001)])
def test_de_parity(problem, N, D):
    gens = 25 if D <= 1000 else 4
    _, resync = _de_parity(problem, N, D, seed=3, gens=gens)
    assert resync <= 2


def test_de_crossover_extremes_and_per_dim_bounds():
    _de_parity("sphere", 16, 9, seed=1, gens=6, CR=0.0)
    _de_parity("sphere", 16, 9, seed=1, gens=6, CR=1.0, F=0.8)
    lb = np.linspace(-5, -1, 13).astype(np.float32)
    ub = np.linspace(1, 5, 13).astype(np.float32)
    de, _ = _de_parity("rastrigin", 24, 13, seed=2, gens=6, lb=lb, ub=ub)
    X, _ = _state(de, 13)
    assert (X >= lb).all() and (X <= ub).all()


def test_de_graphed_equals_stepwise_and_view_neutral():
    N, D, p = 70, 45, "ackley"
    a = ev.DE(N, D, -32.768, 32.768, seed=5)
    a.step(p, 40)
    b = ev.DE(N, D, -32.768, 32.768, seed=5)
    b.step(p, 0)
    for _ in range(40):
        b.step(p, 1)
        b.view("X")  # gathers the population into one buffer: must not change the trajectory
    assert np.array_equal(_state(a, D)[0], _state(b, D)[0])
    assert np.array_equal(a.history(), b.history())
    fa, ia, ra = a.best()
    assert fa == a.view("F").cpu().numpy().min() and np.array_equal(ra, _state(a, D)[0][ia])


@pytest.mark.parametrize("problem,N,D", [("sphere", 3000, 100), ("rosenbrock", 1001, 97),
                                         ("griewank", 777, 250), ("ackley", 5000, 16),
                                         ("rastrigin", 70, 128), ("rosenbrock", 200, 5)])
def test_de_flat_kernel_equals_row_walk(problem, N, D):
    """Rows of <= 256 floats run the flat-tile DE kernel (k_de_gen_flat: donors resolved and
    L2-prefetched per target, the tile's trial quads walked flat, f(u) folded from shared
    memory in the geometry's order) -- bitwise the row-walk kernel (EVOX_FLAG_NO_WAVE)."""
    lb, ub = WL.BOUNDS[problem]
    a = ev.DE(N, D, lb, ub, seed=23)
    a.step(problem, 12)
    b = ev.DE(N, D, lb, ub, seed=23, flags=E.FLAG_NO_WAVE)
    b.step(problem, 12)
    xa, fa = _state(a, D)
    xb, fb = _state(b, D)
    assert np.array_equal(xa, xb) and np.array_equal(fa, fb)
    assert np.array_equal(a.history(), b.history())
    assert a.best()[:2] == b.best()[:2]


@pytest.mark.gpu
@pytest.mark.parametrize("gens", [1, 2, 7])
def test_de_best_row_before_any_gather(gens):
    """best() reads the winning row from whichever of the two buffers holds it (no
    population-wide gather): it must equal the row view("X") gathers afterwards."""
    N, D, p = 300, 37, "rastrigin"
    a = ev.DE(N, D, -5.12, 5.12, seed=11)
    a.step(p, gens)
    fa, ia, ra = a.best()
    X = a.view("X").cpu().numpy()[:, :D]
    F = a.view("F").cpu().numpy()
    assert fa == F.min() and ia == int(np.argmin(F)) and np.array_equal(ra, X[ia])


def test_de_large_population_sampled():
    """pop 2^20 x 100 (past the paper's 16,384 DE limit): one generation,
    sampled targets recomputed one by one by the oracle."""
    N, D, seed, p = 1 << 20, 100, 0, "sphere"
    de = ev.DE(N, D, -5.12, 5.12, seed=seed)
    de.step(p, 0)
    X0 = de.view("X").cpu().numpy()[:, :D].copy()
    f0 = de.view("F").cpu().numpy().copy()
    de.step(p, 1)
    X1 = de.view("X").cpu().numpy()[:, :D]
    f1 = de.view("F").cpu().numpy()
    rng = np.random.default_rng(0)
    for i in rng.integers(0, N, 64):
        r = O.de_indices(N, int(i), 0, seed)
        U = O.draw(1, D, int(i), 0, 10, seed)[0]
        u = O.de_trial_with(X0[i], X0[r[0]], X0[r[1]], X0[r[2]], U, O.de_jrand(D, int(i), 0, seed),
                            0.5, 0.9, -5.12, 5.12)
        fu = float(O.evaluate(p, u[None])[0])
        if near_tie(fu, f0[i]):
            continue
        expect = u if fu <= f0[i] else X0[i]
        assert np.array_equal(X1[i], expect), i
    assert (f1 <= f0).all()


@pytest.mark.parametrize("gens", [10, 100])
def test_de_d1_sampled_generations(gens):
    """D1 (DE/Sphere 1e6 x 100) through the flat-tile kernel the bench times: every generation,
    sampled targets recomputed one by one by the oracle from the GPU's pre-generation
    population (donors, crossover, greedy <= replacement; north_star 10 / 100 generations)."""
    N, D, seed, p = 1_000_000, 100, 0, "sphere"
    de = ev.DE(N, D, -5.12, 5.12, seed=seed)
    de.step(p, 0)
    rng = np.random.default_rng(1)
    for t in range(gens):
        X0 = de.view("X").cpu().numpy()[:, :D].copy()
        f0 = de.view("F").cpu().numpy().copy()
        de.step(p, 1)
        X1 = de.view("X").cpu().numpy()[:, :D]
        f1 = de.view("F").cpu().numpy()
        for i in rng.integers(0, N, 16 if gens > 10 else 64):
            r = O.de_indices(N, int(i), t, seed)
            U = O.draw(1, D, int(i), t, 10, seed)[0]
            u = O.de_trial_with(X0[i], X0[r[0]], X0[r[1]], X0[r[2]], U,
                                O.de_jrand(D, int(i), t, seed), 0.5, 0.9, -5.12, 5.12)
            fu = float(O.evaluate(p, u[None])[0])
            if near_tie(fu, f0[i]):
                continue
            expect = u if fu <= f0[i] else X0[i]
            assert np.array_equal(X1[i], expect), (t, i)
        assert (f1 <= f0).all()
        assert de.history()[-1] == f1.min()
    de.close()


def test_de_config_errors():
    with pytest.raises(E.ConfigError):
        ev.DE(3, 4, -1, 1)
    with pytest.raises(E.InvalidArgument):
        ev.DE(10, 4, -1, 1, CR=1.5)
    for F in (0.0, -0.5, 2.5, float("nan")):  # SPEC de_setup: F in (0, 2]
        with pytest.raises(E.InvalidArgument):
            ev.DE(10, 4, -1, 1, F=F)
    assert ev.DE(10, 4, -1, 1, F=2.0).best(with_row=False)[:2] == (float("inf"), -1)
    assert ev.CSO(16, 4, -1, 1).best(with_row=False)[:2] == (float("inf"), -1)
    de = ev.DE(10, 4, -1, 1)
    de.step("sphere", 1)
    with pytest.raises(E.ContractError):
        de.step("ackley", 1)


# ------------------------------------------------------- sharded DE (peer memory)
def _de_group(W, N, D, lb, ub, seed):
    hs = [ev.DE(N, D, lb, ub, seed=seed, rank=r, world=W, stream=torch.cuda.Stream())
          for r in range(W)]
    bases = [h.state_base() for h in hs]
    for h in hs:
        h.connect_local(bases)
    return hs


@pytest.mark.parametrize("W,N,D,problem", [(2, 64, 37, "ackley"), (3, 50, 100, "sphere"),
                                           (4, 97, 1000, "rastrigin"), (8, 203, 20, "griewank"),
                                           (2, 9, 4099, "rosenbrock")])
def test_de_sharded_equals_single(W, N, D, problem):
    """Donors drawn from the whole population, read across shards through peer memory:
    the sharded trajectory is bitwise the single-shard one."""
    lb, ub = WL.BOUNDS[problem]
    ref = ev.DE(N, D, lb, ub, seed=6)
    ref.step(problem, 30)
    hs = _de_group(W, N, D, lb, ub, 6)
    for h in hs:
        h.step(problem, 0)
    for _ in range(3):
        for h in hs:
            h.step(problem, 10)
    for h in hs:
        h.sync()
    X = np.concatenate([h.view("X").cpu().numpy()[:, :D] for h in hs])
    F = np.concatenate([h.view("F").cpu().numpy() for h in hs])
    assert np.array_equal(X, ref.view("X").cpu().numpy()[:, :D])
    assert np.array_equal(F, ref.view("F").cpu().numpy())
    rb = ref.best()
    for h in hs:
        assert np.array_equal(h.history(), ref.history())
        b = h.best()
        assert b[0] == rb[0] and b[1] == rb[1] and np.array_equal(b[2], rb[2])


def test_de_sharded_requires_connect():
    h = ev.DE(16, 4, -1, 1, rank=0, world=2)
    with pytest.raises(E.ContractError):
        h.step("sphere", 1)


def test_de_save_load_roundtrip():
    N, D, p = 40, 23, "rastrigin"
    a = ev.DE(N, D, -5.12, 5.12, seed=4)
    a.step(p, 6)
    blob = a.save()
    a.step(p, 5)
    b = ev.DE(N, D, -5.12, 5.12, seed=4)
    b.load(blob)
    b.step(p, 5)
    assert np.array_equal(_state(a, D)[0], _state(b, D)[0])
    assert np.array_equal(a.history(), b.history())
    c = ev.DE(N, D, -5.12, 5.12, seed=4, CR=0.5)
    with pytest.raises(E.ContractError):
        c.load(blob)


@pytest.mark.parametrize("algo", ["de", "cso"])
def test_best_from_generation_key_and_after_load(algo):
    """best() of a single-rank CSO / DE reads the minimum key the generation kernel left in the
    control block (no population argmin): it must equal the population's argmin and row; after
    load() (whose control block predates the blob) it recomputes, with the same answer."""
    N, D, p = 500, 29, "ackley"
    mk = (lambda: ev.DE(N, D, -32.768, 32.768, seed=8)) if algo == "de" else \
        (lambda: ev.CSO(N, D, -32.768, 32.768, block=100, seed=8))
    a = mk()
    for g in (0, 1, 5):
        a.step(p, g)
        fa, ia, ra = a.best()
        F = a.view("F").cpu().numpy()
        X = a.view("X").cpu().numpy()[:, :D]
        assert fa == F.min() and ia == int(np.argmin(F)) and np.array_equal(ra, X[ia])
    blob = a.save()
    b = mk()
    b.load(blob)
    assert b.best()[:2] == a.best()[:2]
    assert np.array_equal(b.best()[2], a.best()[2])
