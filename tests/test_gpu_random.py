"""Randomised parity sweep: random problems, shapes (ragged dims, every launch geometry),
seeds and bounds, for PSO, CSO and DE, against the oracle (near-tie protocol R-9)."""
import numpy as np
import pytest

import oracle as O
from parity import assert_fitness, assert_positions, compare_pso, gpu_pso_state, near_tie, \
    resync_oracle_from_gpu

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2301_12457_b200 as ev  # noqa: E402
from paper_2301_12457_b200 import evox as E  # noqa: E402
from paper_2301_12457_b200 import workloads as WL  # noqa: E402
from test_gpu_sharded_oracle import cso_flipped_pairs_are_near_ties  # noqa: E402

PROBLEMS = list(WL.BOUNDS)
_rng = np.random.default_rng(20260417)
CASES = []
for k in range(24):
    D = int(_rng.choice([1, 2, 3, 5, 7, 13, 31, 64, 99, 127, 129, 255, 257, 513, 1021, 2049,
                         4095, 4097, 9001]))
    N = int(_rng.integers(4, 120 if D < 2000 else 12))
    CASES.append((k, PROBLEMS[k % 5], N, D, int(_rng.integers(0, 2 ** 40))))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("k,problem,N,D,seed", CASES)
def test_random_pso(k, problem, N, D, seed):
    lo, hi = WL.BOUNDS[problem]
    if k % 3 == 0:  # per-dimension bounds
        lb = np.linspace(lo, lo / 2, D).astype(np.float32)
        ub = np.linspace(hi / 2, hi, D).astype(np.float32)
    else:
        lb, ub = lo, hi
    pso = ev.PSO(N, D, lb, ub, seed=seed, flags=E.FLAG_NO_SMALL if k % 2 else 0)
    pso.step(problem, 0)
    st = O.pso_run(problem, N, D, lb, ub, seed=seed, n_gens=0)
    g = gpu_pso_state(pso, D)
    if compare_pso(g, st, label="t=0"):
        st = resync_oracle_from_gpu(st, g)
    for t in range(1, 6):
        prev = g["pf"]
        pso.step(problem, 1)
        st = O.pso_run(problem, N, D, lb, ub, seed=seed, n_gens=1, state=st)
        g = gpu_pso_state(pso, D)
        if compare_pso(g, st, prev_pf_gpu=prev, label=f"t={t}"):
            st = resync_oracle_from_gpu(st, g)


@pytest.mark.parametrize("k,problem,N,D,seed", CASES[::2])
def test_random_cso(k, problem, N, D, seed):
    lb, ub = WL.BOUNDS[problem]
    N = N + (N % 2)
    B = int(np.random.default_rng(seed).integers(2, N + 1))
    cso = ev.CSO(N, D, lb, ub, block=B, seed=seed)
    cso.step(problem, 0)
    X, V, f, F64 = O.cso_init(problem, N, D, lb, ub, seed)
    assert np.array_equal(cso.view("X").cpu().numpy()[:, :D], X)
    f = cso.view("F").cpu().numpy().copy()
    resync = 0
    for t in range(4):
        f_prev = f.copy()
        cso.step(problem, 1)
        O.cso_generation(problem, X, V, f, F64, B, t, seed, lb, ub)
        Xg = cso.view("X").cpu().numpy()[:, :D]
        Vg = cso.view("V").cpu().numpy()[:, :D]
        fg = cso.view("F").cpu().numpy()
        if not np.array_equal(Xg, X):
            # a flipped winner decision: only at a near-tie of that pair (R-9), then resync
            cso_flipped_pairs_are_near_ties(Xg, X, f_prev, N, B, t, seed)
            resync += 1
            X, V = Xg.copy(), Vg.copy()
        else:
            assert np.array_equal(Vg, V)
        assert_fitness(fg, O.evaluate(problem, Xg), f"CSO t={t + 1}")
        f = fg.copy()
        F64 = O.evaluate(problem, X)
    assert resync <= 1


@pytest.mark.parametrize("k,problem,N,D,seed", CASES[1::2])
def test_random_de(k, problem, N, D, seed):
    lb, ub = WL.BOUNDS[problem]
    de = ev.DE(N, D, lb, ub, seed=seed)
    de.step(problem, 0)
    X, f, F64 = O.de_init(problem, N, D, lb, ub, seed)
    assert np.array_equal(de.view("X").cpu().numpy()[:, :D], X)
    f = de.view("F").cpu().numpy().copy()
    for t in range(4):
        de.step(problem, 1)
        O.de_generation(problem, X, f, F64, t, seed, lb, ub)
        Xg = de.view("X").cpu().numpy()[:, :D]
        fg = de.view("F").cpu().numpy()
        for i in np.nonzero((Xg != X).any(1))[0]:
            # a flipped accept/reject: the GPU's row and the oracle's row (one of them the
            # trial, the other the target) must be near-tied in fitness
            assert near_tie(float(O.evaluate(problem, Xg[i][None])[0]),
                            float(O.evaluate(problem, X[i][None])[0])), (t, i)
        X = Xg.copy()
        assert_fitness(fg, O.evaluate(problem, Xg), f"DE t={t + 1}")
        f = fg.copy()
        F64 = O.evaluate(problem, X)
