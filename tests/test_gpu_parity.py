"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bars (R-9): Philox words and X0 bit-exact; fitness within
max(1e-5 |F64|, 1e-6); positions within 1e-6 relative (observed bit-exact);
pbest/gbest decisions exact outside near-ties, near-ties re-synchronised and
logged; checkpoints at 1, 10 and 100 generations.
"""
import numpy as np
import pytest

import oracle as O
from parity import (assert_fitness, assert_positions, compare_pso, gpu_pso_state, near_tie,
                    resync_oracle_from_gpu)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2301_12457_b200 as ev  # noqa: E402
from paper_2301_12457_b200 import evox as E  # noqa: E402
from paper_2301_12457_b200 import workloads as WL  # noqa: E402
from test_gpu_sharded_oracle import cso_flipped_pairs_are_near_ties  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


# ------------------------------------------------------------------ Philox
def test_philox_gpu_matches_kat_and_oracle(golden_dir):
    import os
    kat = []
    for line in open(os.path.join(golden_dir, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        kat.append(v)
    for v in kat:
        ctr = torch.tensor(np.array([v[0:4]], np.uint32).view(np.int32), device="cuda")
        out = E.debug_philox(ctr, v[4], v[5]).cpu().numpy().view(np.uint32)[0]
        assert list(out) == v[6:10]
    rng = np.random.default_rng(0)
    C = rng.integers(0, 2 ** 32, (4096, 4), dtype=np.uint64).astype(np.uint32)
    key = (0xDEADBEEF, 0x12345678)
    out = E.debug_philox(torch.tensor(C.view(np.int32), device="cuda"), *key).cpu().numpy()
    out = out.view(np.uint32)
    for i in range(0, 4096, 97):
        assert list(out[i]) == list(O.philox(C[i], key))


# -------------------------------------------------------------------- init
@pytest.mark.parametrize("N,D", [(1, 1), (7, 3), (100, 10), (33, 37), (64, 1000), (5, 4099),
                                 (3, 40001)])
def test_init_bitwise(N, D):
    lb = np.linspace(-3, -1, D).astype(np.float32)
    ub = np.linspace(1, 600, D).astype(np.float32)
    pso = ev.PSO(N, D, lb, ub, seed=1234567890123)
    X = pso.view("X").cpu().numpy()
    V = pso.view("V").cpu().numpy()
    Xo, Vo = O.pso_init(N, D, 0, lb, ub, 1234567890123)
    assert np.array_equal(X[:, :D], Xo)
    assert not X[:, D:].any() and not V.any()
    assert np.array_equal(pso.view("P").cpu().numpy(), X)


# -------------------------------------------------------------------- eval
EVAL_SHAPES = [(1, 1), (3, 2), (5, 3), (64, 4), (100, 10), (37, 33), (130, 100), (9, 257),
               (513, 1000), (16, 1001), (7, 3000), (8, 4099), (3, 40001), (2, 100000)]


@pytest.mark.parametrize("problem", list(WL.BOUNDS))
@pytest.mark.parametrize("N,D", EVAL_SHAPES)
def test_eval_parity(problem, N, D):
    for k, X in enumerate((WL.uniform_rows(N, D, problem, seed=D + N),
                           WL.uniform_rows(N, D, problem, seed=7, scale=1e-2),
                           WL.near_optimum_rows(N, D, problem, seed=3, radius=1e-4))):
        Xp = torch.from_numpy(WL.padded(X)).cuda()
        f = ev.evaluate(problem, Xp, dim=D).cpu().numpy()
        assert_fitness(f, O.evaluate(problem, X), f"{problem} {N}x{D} input {k}")


def test_eval_closed_forms_gpu():
    D = 1003
    z = np.zeros((1, D), np.float32)
    for p in WL.BOUNDS:
        x = z if p != "rosenbrock" else z + 1
        f = ev.evaluate(p, torch.from_numpy(WL.padded(x)).cuda(), dim=D).item()
        assert abs(f) <= 1e-6, (p, f)
    k = np.random.default_rng(1).integers(-5, 6, (4, D)).astype(np.float32)
    f = ev.evaluate("rastrigin", torch.from_numpy(WL.padded(k)).cuda(), dim=D).cpu().numpy()
    assert np.array_equal(f, (k.astype(np.float64) ** 2).sum(1).astype(np.float32))
    f = ev.evaluate("rosenbrock", torch.from_numpy(WL.padded(z)).cuda(), dim=D).item()
    assert f == D - 1


def test_eval_permutation_and_empty():
    X = WL.uniform_rows(300, 57, "griewank", 5)
    perm = np.random.default_rng(2).permutation(300)
    a = ev.evaluate("griewank", torch.from_numpy(WL.padded(X)).cuda(), dim=57).cpu().numpy()
    b = ev.evaluate("griewank", torch.from_numpy(WL.padded(X[perm])).cuda(), dim=57).cpu().numpy()
    assert np.array_equal(a[perm], b)
    e = ev.evaluate("sphere", torch.zeros((0, 8), device="cuda"), dim=5)
    assert e.numel() == 0


# ----------------------------------------------------------------- PSO step
PSO_CASES = [("sphere", 100, 10, -5.12, 5.12, 0),        # C1
             ("ackley", 64, 37, -32.768, 32.768, 1),
             ("rastrigin", 50, 8, -5.12, 5.12, 2),
             ("griewank", 40, 100, -600, 600, 3),
             ("rosenbrock", 33, 101, -5, 10, 4),
             ("rosenbrock", 9, 4099, -5, 10, 5),
             ("griewank", 21, 3000, -600, 600, 7),
             ("rosenbrock", 13, 2999, -5, 10, 8),
             ("ackley", 6, 40001, -32.768, 32.768, 6)]


def _run_parity(problem, N, D, lb, ub, seed, gens, checkpoints=(1, 10, 100), threads=1):
    pso = ev.PSO(N, D, lb, ub, seed=seed)
    pso.step(problem, 0)
    st = O.pso_run(problem, N, D, lb, ub, seed=seed, n_gens=0, threads=threads)
    g = gpu_pso_state(pso, D)
    flips = compare_pso(g, st, label=f"{problem} t=0")
    if flips:
        st = resync_oracle_from_gpu(st, g)
    log = []
    for t in range(1, gens + 1):
        prev_pf = g["pf"]
        pso.step(problem, 1)
        st = O.pso_run(problem, N, D, lb, ub, seed=seed, n_gens=1, state=st, threads=threads)
        g = gpu_pso_state(pso, D)
        flips = compare_pso(g, st, prev_pf_gpu=prev_pf, label=f"{problem} t={t}")
        if flips:
            log.append((t, flips))
            st = resync_oracle_from_gpu(st, g)
        if t in checkpoints:
            # full-state checkpoint (R-9): X, V, P, pf, f, G, gf
            assert_positions(g["X"], st.X, f"checkpoint {t} X")
            assert_positions(g["P"], st.P, f"checkpoint {t} P")
            assert_positions(g["G"], st.G, f"checkpoint {t} G")
            assert_fitness(g["f"], st.F64, f"checkpoint {t} f")
    return pso, log


@pytest.mark.parametrize("problem,N,D,lb,ub,seed", PSO_CASES)
def test_pso_step_parity_100_gens(problem, N, D, lb, ub, seed):
    gens = 100 if D <= 1000 else 10
    pso, log = _run_parity(problem, N, D, lb, ub, seed, gens)
    if log:
        print(f"near-tie resyncs ({problem}): {log}")
    assert len(log) <= gens // 10, log  # near-ties are rare


@pytest.mark.parametrize("problem,N,D,lb,ub,seed", PSO_CASES[:5])
def test_pso_graphed_equals_stepwise(problem, N, D, lb, ub, seed):
    """step(100) in one call (CUDA-graph replay) is bitwise equal to 100 x step(1)."""
    a = ev.PSO(N, D, lb, ub, seed=seed)
    a.step(problem, 100)
    b = ev.PSO(N, D, lb, ub, seed=seed)
    b.step(problem, 0)
    for _ in range(100):
        b.step(problem, 1)
    ga, gb = gpu_pso_state(a, D), gpu_pso_state(b, D)
    for k in ("X", "V", "P", "f", "pf", "G", "hist"):
        assert np.array_equal(ga[k], gb[k]), k
    assert ga["gidx"] == gb["gidx"] and ga["gf"] == gb["gf"]


@pytest.mark.parametrize("problem,N,D,lb,ub,seed", PSO_CASES[:5])
def test_pso_small_kernel_equals_grid_kernel(problem, N, D, lb, ub, seed):
    """The persistent single-CTA kernel (tiny populations) is bitwise identical to the
    multi-CTA generation kernel."""
    a = ev.PSO(N, D, lb, ub, seed=seed)
    a.step(problem, 60)
    b = ev.PSO(N, D, lb, ub, seed=seed, flags=E.FLAG_NO_SMALL)
    b.step(problem, 60)
    ga, gb = gpu_pso_state(a, D), gpu_pso_state(b, D)
    for k in ("X", "V", "P", "f", "pf", "G", "hist"):
        assert np.array_equal(ga[k], gb[k]), k
    assert ga["gidx"] == gb["gidx"] and ga["gf"] == gb["gf"]


@pytest.mark.parametrize("problem,N,D", [("ackley", 10_000, 1000),    # C2, warp per row
                                         ("rosenbrock", 3001, 100),   # 4 lanes per row
                                         ("griewank", 1999, 250),     # 8 lanes per row
                                         ("rastrigin", 21, 5000),     # CTA per row
                                         ("sphere", 700, 1001)])      # ragged tail
def test_pso_mid_kernel_equals_stepwise(problem, N, D):
    """The persistent cooperative kernel (mid-size populations, n generations in one launch,
    grid barrier between generations) is bitwise identical to one k_pso_gen launch per
    generation; two step calls exercise the barrier epoch across launches."""
    lb, ub = WL.BOUNDS[problem]
    a = ev.PSO(N, D, lb, ub, seed=31)
    a.step(problem, 10)
    a.step(problem, 15)
    b = ev.PSO(N, D, lb, ub, seed=31, flags=E.FLAG_NO_MID)
    b.step(problem, 25)
    ga, gb = gpu_pso_state(a, D), gpu_pso_state(b, D)
    for k in ("X", "V", "P", "f", "pf", "G", "hist"):
        assert np.array_equal(ga[k], gb[k]), k
    assert ga["gidx"] == gb["gidx"] and ga["gf"] == gb["gf"]


def test_pso_mid_kernel_interleaved_with_ask_tell():
    """Cooperative launches interleaved with unfused ask/tell generations (other paths advancing
    the population between launches, so the cooperative kernel's per-generation key slots must be
    re-initialised) -- bitwise the same generations all run one launch at a time."""
    N, D, p = 3001, 1000, "ackley"
    lb, ub = WL.BOUNDS[p]
    a = ev.PSO(N, D, lb, ub, seed=19)
    b = ev.PSO(N, D, lb, ub, seed=19, flags=E.FLAG_NO_MID)
    def ask_tell(h):  # evaluated on the handle's stream, so it sees ask's population
        h.tell(ev.evaluate(p, h.ask(), dim=D, stream=h.stream))

    for h in (a, b):
        h.step(p, 3)
        for _ in range(2):  # two unfused generations
            ask_tell(h)
        h.step(p, 4)
        ask_tell(h)
        h.step(p, 2)
    ga, gb = gpu_pso_state(a, D), gpu_pso_state(b, D)
    for k in ("X", "V", "P", "f", "pf", "G", "hist"):
        assert np.array_equal(ga[k], gb[k]), k
    assert ga["gidx"] == gb["gidx"] and ga["gf"] == gb["gf"]


@pytest.mark.parametrize("problem,N,D", [("ackley", 3001, 1000), ("rosenbrock", 3001, 100),
                                         ("rastrigin", 700, 1001), ("griewank", 3001, 1000),
                                         ("sphere", 2401, 257)])
def test_pso_mid_tail_tiles_per_dimension_bounds(problem, N, D):
    """The cooperative kernel's flat tail tiles with per-column bounds (non-uniform-bounds
    instantiation) are bitwise one k_pso_gen launch per generation, inside every column's box."""
    lo, hi = WL.BOUNDS[problem]
    lb = np.linspace(lo, lo / 5, D).astype(np.float32)
    ub = np.linspace(hi / 2, hi, D).astype(np.float32)
    a = ev.PSO(N, D, lb, ub, seed=13)
    a.step(problem, 6)
    a.step(problem, 5)
    b = ev.PSO(N, D, lb, ub, seed=13, flags=E.FLAG_NO_MID)
    b.step(problem, 11)
    ga, gb = gpu_pso_state(a, D), gpu_pso_state(b, D)
    for k in ("X", "V", "P", "f", "pf", "G", "hist"):
        assert np.array_equal(ga[k], gb[k]), k
    assert ga["gidx"] == gb["gidx"] and ga["gf"] == gb["gf"]
    assert (ga["X"] >= lb).all() and (ga["X"] <= ub).all()


@pytest.mark.parametrize("problem,N,D", [("ackley", 400, 100_000), ("rosenbrock", 2000, 17_001),
                                         ("griewank", 800, 50_000), ("ackley", 40_000, 1000),
                                         ("rosenbrock", 34_000, 1001), ("sphere", 9_000, 3999),
                                         # short rows: k_pso_gen_flat (4 / 8 lanes per row)
                                         ("griewank", 340_001, 100), ("rosenbrock", 340_003, 97),
                                         ("ackley", 140_000, 250), ("sphere", 600_000, 60),
                                         ("rastrigin", 2_100_003, 16), ("rosenbrock", 400_001, 128)])
def test_pso_wave_kernel_equals_persistent(problem, N, D):
    """Big populations (> 2^25 elements) with rows of > 128 floats run the wave grid
    (k_pso_gen_wave: one CTA per row block, fewer chunks in flight, more CTAs/SM, gbest
    published by k_pso_fin) -- bitwise the persistent grid-stride kernel (EVOX_FLAG_NO_WAVE):
    same per-row code and reduction order."""
    lb, ub = WL.BOUNDS[problem]
    a = ev.PSO(N, D, lb, ub, seed=17)
    a.step(problem, 4)
    b = ev.PSO(N, D, lb, ub, seed=17, flags=E.FLAG_NO_WAVE)
    b.step(problem, 4)
    ga, gb = gpu_pso_state(a, D), gpu_pso_state(b, D)
    for k in ("X", "V", "P", "f", "pf", "G", "hist"):
        assert np.array_equal(ga[k], gb[k]), k
    assert ga["gidx"] == gb["gidx"] and ga["gf"] == gb["gf"]
    a.close()
    b.close()


@pytest.mark.parametrize("problem,N,D", [("ackley", 340_001, 100), ("rosenbrock", 140_000, 250),
                                         ("griewank", 400_000, 90), ("ackley", 40_000, 1000),
                                         ("rastrigin", 4_000, 9000)])
def test_pso_flat_kernel_per_dimension_bounds(problem, N, D):
    """The flat-tile kernel and the wave kernels (warp per row with the tile prefetch, CTA per
    row) with per-column bounds (the non-uniform-bounds instantiations) are bitwise the
    persistent row walk, and every position stays inside its column's box."""
    lo, hi = WL.BOUNDS[problem]
    lb = np.linspace(lo, lo / 4, D).astype(np.float32)
    ub = np.linspace(hi / 3, hi, D).astype(np.float32)
    a = ev.PSO(N, D, lb, ub, seed=5)
    a.step(problem, 3)
    b = ev.PSO(N, D, lb, ub, seed=5, flags=E.FLAG_NO_WAVE)
    b.step(problem, 3)
    ga, gb = gpu_pso_state(a, D), gpu_pso_state(b, D)
    for k in ("X", "V", "P", "f", "pf", "G", "hist"):
        assert np.array_equal(ga[k], gb[k]), k
    assert (ga["X"] >= lb).all() and (ga["X"] <= ub).all()
    a.close()
    b.close()


def test_pso_wave_kernel_peer_group():
    """The wave grid with the in-kernel peer exchange (k_pso_fin runs it), W = 2 ranks of
    4e7 elements each (CTA-per-row geometry), bitwise the single-shard persistent run."""
    N, D, p = 800, 100_000, "ackley"
    ref = ev.PSO(N, D, -32.768, 32.768, seed=2, flags=E.FLAG_NO_WAVE)
    ref.step(p, 3)
    hs = [ev.PSO(N, D, -32.768, 32.768, seed=2, rank=r, world=2, stream=torch.cuda.Stream())
          for r in range(2)]
    boxes = [h.mailbox()[0] for h in hs]
    for h in hs:
        h.connect_local(boxes)
    for h in hs:
        h.step(p, 3)
    for h in hs:
        h.sync()
    X = np.concatenate([h.view("X").cpu().numpy() for h in hs])
    assert np.array_equal(X, ref.view("X").cpu().numpy())
    for h in hs:
        assert h.best()[:2] == ref.best()[:2]
        assert np.array_equal(h.history(), ref.history())


@pytest.mark.parametrize("problem,N,D", [("ackley", 300, 1000), ("rosenbrock", 77, 1001),
                                         ("griewank", 64, 4096), ("rastrigin", 130, 600),
                                         ("sphere", 1000, 300)])
def test_pso_tma_kernel_equals_ldg_kernel(problem, N, D):
    """The TMA-staged generation kernel (opt-in, warp-per-row geometry) is bitwise identical
    to the default LDG kernel."""
    lb, ub = WL.BOUNDS[problem]
    a = ev.PSO(N, D, lb, ub, seed=12, flags=E.FLAG_NO_SMALL | E.FLAG_TMA)
    a.step(problem, 9)
    b = ev.PSO(N, D, lb, ub, seed=12, flags=E.FLAG_NO_SMALL)
    b.step(problem, 9)
    ga, gb = gpu_pso_state(a, D), gpu_pso_state(b, D)
    for k in ("X", "V", "P", "f", "pf", "G", "hist"):
        assert np.array_equal(ga[k], gb[k]), k


def test_pso_c1_oneshot_matches_oracle():
    """C1 (PSO/Sphere 100x10, 100 generations, seed 0) in one step(100) call."""
    pso = ev.PSO(100, 10, -5.12, 5.12, seed=0)
    pso.step("sphere", 100)
    st = O.pso_run("sphere", 100, 10, -5.12, 5.12, seed=0, n_gens=100)
    g = gpu_pso_state(pso, 10)
    assert_positions(g["X"], st.X, "C1 X")
    assert_fitness(g["hist"], np.asarray(st.hist, np.float64), "C1 hist")
    assert g["gidx"] == st.gidx
    assert g["gf"] < 1e-4  # S:321-style convergence on the GPU as well


def test_pso_ask_tell_equals_step():
    """Unfused ask/evaluate/tell produces the same state as fused step (bitwise)."""
    N, D, p = 70, 45, "ackley"
    a = ev.PSO(N, D, -32.768, 32.768, seed=11)
    a.step(p, 12)
    b = ev.PSO(N, D, -32.768, 32.768, seed=11)
    for _ in range(13):
        X = b.ask()
        f = ev.evaluate(p, X, dim=D, stream=b.stream)
        b.tell(f)
    ga, gb = gpu_pso_state(a, D), gpu_pso_state(b, D)
    for k in ("X", "V", "P", "f", "pf", "G", "hist"):
        assert np.array_equal(ga[k], gb[k]), k


def test_pso_ask_tell_external_fitness_vs_oracle():
    """tell() with caller fitness (here: a shifted Sphere computed by torch) follows the
    oracle's tell/move primitives."""
    N, D, seed = 40, 12, 5
    pso = ev.PSO(N, D, -2, 2, seed=seed)
    X, V = O.pso_init(N, D, 0, -2, 2, seed)
    P, pf = X.copy(), np.full(N, np.inf, np.float32)
    G, gf = np.zeros(D, np.float32), np.inf
    for t in range(6):
        Xg = pso.ask()
        assert np.array_equal(Xg.cpu().numpy()[:, :D], X), t
        fx = ((Xg[:, :D] - 0.25) ** 2).sum(1).contiguous()
        pso.tell(fx)
        f = fx.cpu().numpy()
        O.pso_tell_rows(X, f, P, pf)
        i, m = O.argmin(f)
        if m < gf:
            gf, G = m, X[i].copy()
        O.pso_move(X, V, P, G, 0, t, seed, 0.6, 2.5, 0.8, -2, 2)
    b = pso.best()
    assert b[0] == gf and np.array_equal(b[2], G)


def test_pso_contract_errors():
    pso = ev.PSO(16, 8, -1, 1, seed=0)
    with pytest.raises(E.ContractError):
        pso.tell(torch.zeros(16, device="cuda"))
    pso.ask()
    with pytest.raises(E.ContractError):
        pso.ask()
    with pytest.raises(E.ContractError):
        pso.step("sphere", 1)
    pso.tell(torch.zeros(16, device="cuda"))
    pso.step("sphere", 2)
    with pytest.raises(E.ContractError):
        pso.step("ackley", 1)
    with pytest.raises(E.InvalidArgument):
        pso.step("sphere", -1)


def test_pso_save_load_roundtrip():
    N, D, p = 64, 33, "rastrigin"
    a = ev.PSO(N, D, -5.12, 5.12, seed=9)
    a.step(p, 5)
    blob = a.save()
    a.step(p, 7)
    b = ev.PSO(N, D, -5.12, 5.12, seed=9)
    b.load(blob)
    b.step(p, 7)
    ga, gb = gpu_pso_state(a, D), gpu_pso_state(b, D)
    for k in ("X", "V", "P", "f", "pf", "G", "hist"):
        assert np.array_equal(ga[k], gb[k]), k
    c = ev.PSO(N, D, -5.12, 5.12, seed=10)
    with pytest.raises(E.ContractError):
        c.load(blob)


def test_pso_view_p_materialise_is_neutral():
    """Reading P (materialising lazy pbest rows) does not change later generations."""
    N, D, p = 48, 20, "griewank"
    a = ev.PSO(N, D, -600, 600, seed=4)
    b = ev.PSO(N, D, -600, 600, seed=4)
    for _ in range(8):
        a.step(p, 1)
        b.step(p, 1)
        b.view("P")
    ga, gb = gpu_pso_state(a, D), gpu_pso_state(b, D)
    for k in ("X", "V", "P", "f", "pf", "G"):
        assert np.array_equal(ga[k], gb[k]), k


def test_pso_user_stream_and_workspace():
    N, D, p = 128, 64, "sphere"
    s = torch.cuda.Stream()
    ws = torch.empty(ev.PSO.workspace_bytes(N, D), dtype=torch.uint8, device="cuda")
    a = ev.PSO(N, D, -5.12, 5.12, seed=3, stream=s, workspace=ws)
    a.step(p, 10)
    b = ev.PSO(N, D, -5.12, 5.12, seed=3)
    b.step(p, 10)
    assert np.array_equal(gpu_pso_state(a, D)["X"], gpu_pso_state(b, D)["X"])
    assert a.info()["stream"] == s.cuda_stream


def test_pso_nccl_exchange_path_single_rank():
    """EVOX_FLAG_FORCE_NCCL: the multi-GPU exchange (record all-gather + gbest select) on a
    1-rank communicator gives the same trajectory bitwise as the direct path."""
    N, D, p = 96, 50, "ackley"
    a = ev.PSO(N, D, -32.768, 32.768, seed=21)
    a.step(p, 15)
    b = ev.PSO(N, D, -32.768, 32.768, seed=21, flags=E.FLAG_FORCE_NCCL)
    b.step(p, 15)
    ga, gb = gpu_pso_state(a, D), gpu_pso_state(b, D)
    for k in ("X", "V", "P", "f", "pf", "G", "hist"):
        assert np.array_equal(ga[k], gb[k]), k
    assert ga["gidx"] == gb["gidx"]


# ---------------------------------------------------- full-size sampled checks
def _sampled_generations_check(problem, N, D, seed, gens=10, n_sample=256, threads=8):
    """At full size, stepped from identical states (north_star: 1 and 10 generations):
    generation 0, then every generation re-derive sampled rows one by one with the oracle
    from the GPU's PRE-move state (X, V, materialised pbest P, gbest G, t) -- positions and
    velocities bitwise, fitness within tolerance, the pbest decision of each sampled row --
    and check the tell on the whole population (gbest strict improvement, lowest index,
    hist)."""
    lb, ub = WL.BOUNDS[problem]
    pso = ev.PSO(N, D, lb, ub, seed=seed)
    pso.step(problem, 0)
    rng = np.random.default_rng(seed)
    rows = np.unique(np.concatenate([[0, N - 1], rng.integers(0, N, n_sample)]))
    ridx = torch.from_numpy(rows).cuda()
    take = lambda k: pso.view(k)[ridx].cpu().numpy()[:, :D].copy()  # noqa: E731
    f0 = pso.view("F").cpu().numpy()
    gf, gi, grow = pso.best()
    m = f0.min()
    assert gf == m and gi == int(np.nonzero(f0 == m)[0][0])
    assert np.array_equal(grow, pso.view("X")[gi].cpu().numpy()[:D])
    assert_fitness(f0[rows], O.evaluate(problem, take("X"), threads), "gen0 sampled f")
    for t in range(gens):
        X0, V0, P0 = take("X"), take("V"), take("P")
        pf0 = pso.view("PF")[ridx].cpu().numpy().copy()
        G0 = pso.view("G").cpu().numpy()[:D].copy()
        gf0 = pso.best(with_row=False)[0]
        pso.step(problem, 1)
        X1, V1, P1 = take("X"), take("V"), take("P")
        f1 = pso.view("F").cpu().numpy()
        pf1 = pso.view("PF")[ridx].cpu().numpy()
        x, v = X0.copy(), V0.copy()
        for k, r in enumerate(rows):
            O.pso_move(x[k:k + 1], v[k:k + 1], P0[k:k + 1], G0, int(r), t, seed, WL.W, WL.PHI_P,
                       WL.PHI_G, lb, ub)
        assert np.array_equal(X1, x), f"t={t + 1}: sampled X"
        assert np.array_equal(V1, v), f"t={t + 1}: sampled V"
        F64 = O.evaluate(problem, X1, threads)
        assert_fitness(f1[rows], F64, f"t={t + 1}: sampled f")
        for k, r in enumerate(rows):  # pbest (S:316 strict), unless a near-tie
            imp = f1[r] < pf0[k]
            if near_tie(f1[r], pf0[k]):
                continue
            assert np.array_equal(P1[k], X1[k] if imp else P0[k]), (t, r)
            assert pf1[k] == (f1[r] if imp else pf0[k]), (t, r)
        gf1, gi1, grow1 = pso.best()
        m = f1.min()
        if m < gf0:  # strict improvement, lowest index among equal minima
            assert gf1 == m and gi1 == int(np.nonzero(f1 == m)[0][0])
            assert np.array_equal(grow1, pso.view("X")[gi1].cpu().numpy()[:D])
        else:
            assert gf1 == gf0
        h = pso.history()
        assert len(h) == t + 2 and h[-1] == m
    pso.close()


@pytest.mark.parametrize("cfg", ["C2", "C4g", "C4r", "C5", "H"])
def test_full_size_sampled_10_gens(cfg):
    c = WL.CONFIGS[cfg]
    free, _ = torch.cuda.mem_get_info()
    need = 3 * c.pop * WL.round4(c.dim) * 4 * 1.1
    if need > free:
        pytest.skip("not enough device memory")
    _sampled_generations_check(c.problem, c.pop, c.dim, seed=0, gens=10,
                               n_sample=64 if c.dim > 10_000 else 256)


@pytest.mark.parametrize("cfg", ["C4g", "C4r", "H", "C2"])
def test_full_size_sampled_100_gens(cfg):
    """north_star's 100-generation comparison at the full-size configs, through the kernels the
    bench times (flat tiles, the prefetching wave grid, the cooperative kernel): every one of
    100 generations, sampled rows re-derived by the oracle from the GPU's pre-move state."""
    c = WL.CONFIGS[cfg]
    free, _ = torch.cuda.mem_get_info()
    need = 3 * c.pop * WL.round4(c.dim) * 4 * 1.1
    if need > free:
        pytest.skip("not enough device memory")
    _sampled_generations_check(c.problem, c.pop, c.dim, seed=3, gens=100, n_sample=96)


def test_c2_full_parity_10_gens():
    """C2 (PSO/Ackley 1e4 x 1000) compared element by element every generation for 10
    generations (near-tie protocol R-9), checkpoints at 1 and 10."""
    c = WL.CONFIGS["C2"]
    lb, ub = WL.BOUNDS[c.problem]
    pso, log = _run_parity(c.problem, c.pop, c.dim, lb, ub, 0, 10, checkpoints=(1, 10),
                           threads=8)
    if log:
        print(f"C2 near-tie resyncs: {log}")
    assert sum(len(f) for _, f in log) <= 20, log


# ------------------------------------------------------------------- CSO
def _cso_parity(problem, N, D, B, seed, gens, phi=0.0):
    lb, ub = WL.BOUNDS[problem]
    cso = ev.CSO(N, D, lb, ub, phi=phi, block=B, seed=seed)
    cso.step(problem, 0)
    X, V, f, F64 = O.cso_init(problem, N, D, lb, ub, seed)
    hist = [float(f.min())]
    resync = 0
    for t in range(gens):
        f_prev = f.copy()
        cso.step(problem, 1)
        O.cso_generation(problem, X, V, f, F64, B, t, seed, lb, ub, phi=phi)
        hist.append(float(f.min()))
        Xg = cso.view("X").cpu().numpy()[:, :D]
        Vg = cso.view("V").cpu().numpy()[:, :D]
        fg = cso.view("F").cpu().numpy()
        if not np.array_equal(Xg, X):
            # a flipped winner: only at a near-tie of the pair (R-9) -- then adopt the GPU state
            cso_flipped_pairs_are_near_ties(Xg, X, f_prev, N, B, t, seed)
            resync += 1
            X, V, f = Xg.copy(), Vg.copy(), fg.copy()
            F64 = O.evaluate(problem, X)
            continue
        assert np.array_equal(Vg, V)
        assert_fitness(fg, O.evaluate(problem, Xg), f"CSO t={t + 1} f")
        f = fg.copy()  # decisions use the GPU's fp32 fitness from here on
    h = cso.history()
    assert len(h) == gens + 1
    assert (np.diff(h) <= 0).all()  # min f is non-increasing (winners are kept)
    return resync


@pytest.mark.parametrize("problem,N,D,B", [("rastrigin", 64, 33, 8), ("sphere", 100, 10, 100),
                                           ("ackley", 50, 100, 16), ("griewank", 33, 7, 33),
                                           ("rosenbrock", 40, 4099, 10)])
def test_cso_parity(problem, N, D, B):
    resync = _cso_parity(problem, N, D, B, seed=3, gens=20 if D < 1000 else 4)
    assert resync <= 2


def test_cso_phi_nonzero_parity():
    assert _cso_parity("sphere", 64, 20, 16, seed=5, gens=10, phi=0.1) <= 1


@pytest.mark.parametrize("problem,N,D,B,phi", [("rastrigin", 3000, 37, 3000, 0.3),
                                               ("griewank", 1030, 130, 10, 0.05)])
def test_cso_phi_nonzero_parity_many_chunks(problem, N, D, B, phi):
    """x-bar over several 256-row chunks / CTAs (R-15 fixed-point sums) vs the oracle's
    fp64 column mean."""
    assert _cso_parity(problem, N, D, B, seed=11, gens=6, phi=phi) <= 1


def test_cso_phi_nccl_path_single_rank():
    N, D, p = 256, 40, "ackley"
    a = ev.CSO(N, D, -32.768, 32.768, phi=0.2, block=32, seed=8)
    a.step(p, 12)
    b = ev.CSO(N, D, -32.768, 32.768, phi=0.2, block=32, seed=8, flags=E.FLAG_FORCE_NCCL)
    b.step(p, 12)
    assert np.array_equal(a.view("X").cpu().numpy(), b.view("X").cpu().numpy())
    assert np.array_equal(a.history(), b.history())


def test_cso_nccl_path_single_rank():
    N, D, p = 128, 40, "rastrigin"
    a = ev.CSO(N, D, -5.12, 5.12, block=16, seed=8)
    a.step(p, 12)
    b = ev.CSO(N, D, -5.12, 5.12, block=16, seed=8, flags=E.FLAG_FORCE_NCCL)
    b.step(p, 12)
    assert np.array_equal(a.view("X").cpu().numpy(), b.view("X").cpu().numpy())
    assert np.array_equal(a.history(), b.history())
    assert a.best()[:2] == b.best()[:2]


@pytest.mark.parametrize("gens", [10, 100])
def test_cso_c3_sampled_gens(gens):
    """C3 (CSO/Rastrigin 1e5 x 1000, B = pop/8): 10 and 100 generations; every generation
    sampled pairs are recomputed one by one by the oracle from the GPU's pre-generation state
    (winner bitwise unchanged, loser update bitwise, loser fitness within tolerance)."""
    c = WL.CONFIGS["C3"]
    lb, ub = WL.BOUNDS[c.problem]
    B = c.pop // 8
    cso = ev.CSO(c.pop, c.dim, lb, ub, block=B, seed=0)
    cso.step(c.problem, 0)
    rng = np.random.default_rng(0)
    for t in range(gens):
        X0 = cso.view("X").cpu().numpy()[:, :c.dim].copy()
        V0 = cso.view("V").cpu().numpy()[:, :c.dim].copy()
        f0 = cso.view("F").cpu().numpy().copy()
        cso.step(c.problem, 1)
        X1 = cso.view("X").cpu().numpy()[:, :c.dim]
        V1 = cso.view("V").cpu().numpy()[:, :c.dim]
        f1 = cso.view("F").cpu().numpy()
        changed = (X1 != X0).any(1)
        assert changed.sum() <= c.pop // 2
        for blk in rng.choice(8, 2, replace=False):
            pairs = O.cso_pairs(B, int(blk), t, 0)
            for a, b in pairs[rng.integers(0, len(pairs), 8 if gens <= 10 else 2)]:
                i, k = blk * B + a, blk * B + b
                if near_tie(f0[i], f0[k]):
                    continue
                w, l = (i, k) if (f0[i] < f0[k] or (f0[i] == f0[k] and i < k)) else (k, i)
                assert np.array_equal(X1[w], X0[w]) and np.array_equal(V1[w], V0[w])
                xl, vl = X0[l].copy(), V0[l].copy()
                R1 = O.draw(1, c.dim, int(l), t, 5, 0)[0]
                R2 = O.draw(1, c.dim, int(l), t, 6, 0)[0]
                O.cso_loser_update_with(X0[w], xl, vl, R1, R2, lb=lb, ub=ub)
                assert np.array_equal(X1[l], xl) and np.array_equal(V1[l], vl), (t, l)
                assert_fitness(f1[[l]], O.evaluate(c.problem, xl[None]), f"C3 t={t + 1} f")
        assert (f1[~changed] == f0[~changed]).all()
        assert cso.history()[-1] == f1.min() <= f0.min()


# ------------------------------------------------------------- edge cases
@pytest.mark.parametrize("problem,N,D", [("ackley", 40, 37), ("rosenbrock", 33, 101),
                                         ("griewank", 9, 1003), ("sphere", 5, 4099)])
def test_pso_per_dimension_bounds(problem, N, D):
    """Non-uniform bounds take the per-column bounds kernel path (UNI=false)."""
    lo, hi = WL.BOUNDS[problem]
    lb = np.linspace(lo, lo / 2, D).astype(np.float32)
    ub = np.linspace(hi / 3, hi, D).astype(np.float32)
    pso, log = _run_parity_bounds(problem, N, D, lb, ub, seed=31, gens=12)
    assert len(log) <= 2, log


def _run_parity_bounds(problem, N, D, lb, ub, seed, gens):
    pso = ev.PSO(N, D, lb, ub, seed=seed)
    pso.step(problem, 0)
    st = O.pso_run(problem, N, D, lb, ub, seed=seed, n_gens=0)
    g = gpu_pso_state(pso, D)
    compare_pso(g, st, label="t=0")
    log = []
    for t in range(1, gens + 1):
        prev_pf = g["pf"]
        pso.step(problem, 1)
        st = O.pso_run(problem, N, D, lb, ub, seed=seed, n_gens=1, state=st)
        g = gpu_pso_state(pso, D)
        assert (g["X"] >= lb).all() and (g["X"] <= ub).all()
        flips = compare_pso(g, st, prev_pf_gpu=prev_pf, label=f"t={t}")
        if flips:
            log.append((t, flips))
            st = resync_oracle_from_gpu(st, g)
    return pso, log


@pytest.mark.parametrize("N,D", [(1, 1), (1, 7), (2, 1), (3, 5), (1, 1000)])
def test_pso_degenerate_sizes(N, D):
    for flags in (0, E.FLAG_NO_SMALL):
        pso = ev.PSO(N, D, -2, 2, seed=4, flags=flags)
        pso.step("rastrigin", 9)
        st = O.pso_run("rastrigin", N, D, -2, 2, seed=4, n_gens=9)
        g = gpu_pso_state(pso, D)
        assert_positions(g["X"], st.X, f"N={N} D={D} X")
        assert_fitness(g["hist"], np.asarray(st.hist, np.float64), "hist")
        assert g["gidx"] == st.gidx


def test_pso_tell_nan_and_signed_zero():
    """R-5 through the unfused tell: NaN never improves and ranks as +inf; -0 ranks as +0,
    ties go to the lowest global index."""
    pso = ev.PSO(6, 4, -1, 1, seed=0)
    pso.ask()
    fit = torch.tensor([float("nan"), 0.0, -0.0, 3.0, float("nan"), -0.0], device="cuda")
    pso.tell(fit)
    f, i, row = pso.best()
    assert f == 0.0 and i == 1
    X0 = pso.view("X").cpu().numpy()[1, :4]
    assert np.array_equal(row, X0)
    pf = pso.view("PF").cpu().numpy()
    assert np.isinf(pf[0]) and np.isinf(pf[4]) and pf[3] == 3.0
    pso.ask()
    pso.tell(torch.full((6,), float("nan"), device="cuda"))
    f2, i2, _ = pso.best()
    assert f2 == 0.0 and i2 == 1  # a NaN generation never replaces gbest
    h = pso.history()
    assert h[0] == 0.0 and np.isinf(h[1])


@pytest.mark.parametrize("N,B,D", [(50, 16, 9), (65, 13, 20), (100, 7, 33), (64, 64, 1001)])
def test_cso_ragged_blocks(N, B, D):
    assert _cso_parity("ackley", N, D, B, seed=11, gens=8) <= 1


def test_cso_per_dimension_bounds():
    N, D, B = 64, 21, 16
    lb = np.linspace(-5.12, -1, D).astype(np.float32)
    ub = np.linspace(1, 5.12, D).astype(np.float32)
    cso = ev.CSO(N, D, lb, ub, block=B, seed=6)
    cso.step("sphere", 5)
    X, V, f, F64 = O.cso_init("sphere", N, D, lb, ub, 6)
    for t in range(5):
        O.cso_generation("sphere", X, V, f, F64, B, t, 6, lb, ub)
    Xg = cso.view("X").cpu().numpy()[:, :D]
    assert np.array_equal(Xg, X)
    assert (Xg >= lb).all() and (Xg <= ub).all()


def test_eval_nonfinite_rows():
    """Non-finite inputs give non-finite fitness; other rows are unaffected."""
    X = WL.uniform_rows(4, 12, "sphere", 1)
    X[1, 3] = np.inf
    X[2, 0] = np.nan
    f = ev.evaluate("sphere", torch.from_numpy(WL.padded(X)).cuda(), dim=12).cpu().numpy()
    assert np.isinf(f[1]) and np.isnan(f[2])
    ref = O.evaluate("sphere", X[[0, 3]])
    assert_fitness(f[[0, 3]], ref, "finite rows")


# ------------------------------------------- CSO global pairing across shards
def _cso_group(W, N, D, lb, ub, B, seed, phi=0.0):
    hs = [ev.CSO(N, D, lb, ub, phi=phi, block=B, seed=seed, rank=r, world=W,
                 stream=torch.cuda.Stream()) for r in range(W)]
    bases = [h.state_base() for h in hs]
    for h in hs:
        h.connect_local(bases)
    return hs


@pytest.mark.parametrize("W,N,D,B,problem", [(2, 64, 33, 64, "rastrigin"),
                                             (3, 50, 100, 50, "ackley"),
                                             (4, 97, 1000, 30, "sphere"),
                                             (8, 203, 20, 203, "griewank"),
                                             (2, 10, 4099, 7, "rosenbrock")])
def test_cso_global_pairing_sharded_equals_single(W, N, D, B, problem):
    """Pairing blocks straddle shards (B = pop is global pairing): losers are updated by
    their owner from winner rows read through peer memory -- bitwise the W = 1 run."""
    lb, ub = WL.BOUNDS[problem]
    ref = ev.CSO(N, D, lb, ub, block=B, seed=4)
    ref.step(problem, 25)
    hs = _cso_group(W, N, D, lb, ub, B, 4)
    for h in hs:
        h.step(problem, 0)
    for _ in range(5):
        for h in hs:
            h.step(problem, 5)
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


@pytest.mark.parametrize("W,N,D,B,problem", [(2, 64, 33, 16, "rastrigin"),
                                             (3, 600, 100, 600, "ackley"),
                                             (4, 1024, 20, 128, "sphere"),
                                             (8, 203, 1000, 203, "griewank")])
def test_cso_phi_sharded_equals_single(W, N, D, B, problem):
    """phi != 0 with W > 1: each rank sums its rows' fixed-point
    column limbs, the ranks exchange them through peer memory every generation, and the
    x-bar -- hence the whole trajectory -- is bitwise the W = 1 run (R-15)."""
    lb, ub = WL.BOUNDS[problem]
    ref = ev.CSO(N, D, lb, ub, phi=0.15, block=B, seed=6)
    ref.step(problem, 12)
    hs = _cso_group(W, N, D, lb, ub, B, 6, phi=0.15)
    for h in hs:
        h.step(problem, 0)
    for _ in range(3):
        for h in hs:
            h.step(problem, 4)
    for h in hs:
        h.sync()
    X = np.concatenate([h.view("X").cpu().numpy()[:, :D] for h in hs])
    assert np.array_equal(X, ref.view("X").cpu().numpy()[:, :D])
    for h in hs:
        assert np.array_equal(h.history(), ref.history())


def test_cso_straddling_blocks_require_connect():
    h = ev.CSO(30, 4, -1, 1, block=30, rank=0, world=2)
    with pytest.raises(E.ContractError):
        h.step("sphere", 1)


@pytest.mark.parametrize("problem,N,D", [("ackley", 200, 1000), ("rosenbrock", 300, 100),
                                         ("griewank", 50, 4099), ("rastrigin", 70, 37),
                                         ("sphere", 9, 40001)])
def test_fused_fitness_equals_evaluate(problem, N, D):
    """the fitness the fused generation kernel computes from registers is
    bitwise the standalone Problem.evaluate of the same population (same per-row
    reduction order: a function of dim only) -- for CSO whenever its row geometry is
    evaluate's (else within the fitness tolerance)."""
    lb, ub = WL.BOUNDS[problem]
    pso = ev.PSO(N, D, lb, ub, seed=1, flags=E.FLAG_NO_SMALL)
    pso.step(problem, 3)
    X = pso.view("X")
    f = ev.evaluate(problem, X.clone(), dim=D).cpu().numpy()
    assert np.array_equal(f, pso.view("F").cpu().numpy())
    cso = ev.CSO(N + N % 2, D, lb, ub, seed=1)
    cso.step(problem, 2)
    f = ev.evaluate(problem, cso.view("X").clone(), dim=D).cpu().numpy()
    if 64 < (D + 3) // 4 <= 1024:
        # the CSO generation walks these rows with 8 lanes per row (evaluate: a warp per
        # row), so only the reduction order differs: equal within the fitness tolerance
        fc = cso.view("F").cpu().numpy()
        assert (np.abs(fc - f) <= np.maximum(1e-5 * np.abs(f), 1e-6)).all()
    else:
        assert np.array_equal(f, cso.view("F").cpu().numpy())
    de = ev.DE(N, D, lb, ub, seed=1)
    de.step(problem, 2)
    f = ev.evaluate(problem, de.view("X").clone(), dim=D).cpu().numpy()
    assert np.array_equal(f, de.view("F").cpu().numpy())


@pytest.mark.parametrize("N,D", [(8, 4099), (3, 40001), (5, 100000)])
def test_griewank_table_equals_per_element(N, D):
    """evox_eval's global Griewank column table (CTA-per-row geometry, ld > 4096) holds
    griewank_h(j) itself: bitwise the per-element computation it replaces."""
    X = torch.from_numpy(WL.padded(WL.uniform_rows(N, D, "griewank", seed=D))).cuda()
    a = ev.evaluate("griewank", X, dim=D).cpu().numpy()
    b = ev.evaluate("griewank", X, dim=D, flags=E.EVAL_NO_HTAB).cpu().numpy()
    assert np.array_equal(a, b)
    assert_fitness(a, O.evaluate("griewank", X.cpu().numpy()[:, :D]), f"griewank {N}x{D}")
