"""Every W > 1 path against the CPU ORACLE (not against the GPU W = 1 run).

The paper's distributed step is "every node evaluates its shard, the results are
all-gathered, one unified tell" (§V-B; SPMD P:571-573)
requires the same result for every W.  The oracle implements that step with W simulated
contiguous shards (oracle_pso_run(W), R-11), and CSO/DE generations whose pairs / donors
span the whole population.  Here W ranks are W handles of one process on one GPU (each on
its own stream; mailboxes / states connected by pointer), or W processes connected through
CUDA IPC, compared element by element every generation with the near-tie protocol (R-9):
a decision may flip only where the two fitness values are within the tolerance, the flip
is re-synchronised, and the number of flips is bounded.
"""
import os

import numpy as np
import pytest

import oracle as O
from parity import (assert_fitness, assert_positions, compare_pso, near_tie,
                    resync_oracle_from_gpu)

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


# ------------------------------------------------------------------ PSO
def _pso_group(W, N, D, lb, ub, seed, **kw):
    hs = [ev.PSO(N, D, lb, ub, seed=seed, rank=r, world=W, stream=torch.cuda.Stream(), **kw)
          for r in range(W)]
    boxes = [h.mailbox()[0] for h in hs]
    for h in hs:
        h.connect_local(boxes)
    return hs


def _sharded_pso_state(hs, D):
    """The whole population's state gathered from the W shards; G, gf, gidx and the
    history from every rank (they must agree: the exchange is replicated)."""
    for h in hs:
        h.sync()
    cat = lambda k: np.concatenate([h.view(k).cpu().numpy() for h in hs])  # noqa: E731
    X, V, P = (cat(k)[:, :D].copy() for k in ("X", "V", "P"))
    G = hs[0].view("G").cpu().numpy()[:D].copy()
    gf, gidx, _ = hs[0].best(with_row=False)
    hist = hs[0].history()
    for h in hs[1:]:
        assert np.array_equal(h.view("G").cpu().numpy()[:D], G)
        assert h.best(with_row=False)[:2] == (gf, gidx)
        assert np.array_equal(h.history(), hist)
    return dict(X=X, V=V, P=P, f=cat("F").copy(), pf=cat("PF").copy(), G=G, gf=gf, gidx=gidx,
                hist=hist)


@pytest.mark.parametrize("W,N,D,problem", [(2, 64, 37, "ackley"), (3, 50, 100, "rosenbrock"),
                                           (4, 97, 300, "rastrigin"), (8, 203, 20, "griewank"),
                                           (2, 9, 4099, "sphere"), (8, 1000, 64, "ackley")])
def test_pso_peer_exchange_vs_oracle(W, N, D, problem):
    """The in-kernel peer-memory exchange (A13, NEXT #1) against oracle_pso_run(W): every
    generation, X, V, P, pf, f, G, gf, gidx and hist of the concatenated shards."""
    lb, ub = WL.BOUNDS[problem]
    seed, gens = 5, 20
    hs = _pso_group(W, N, D, lb, ub, seed)
    for h in hs:
        h.step(problem, 0)
    st = O.pso_run(problem, N, D, lb, ub, seed=seed, n_gens=0, W=W)
    g = _sharded_pso_state(hs, D)
    flips = compare_pso(g, st, label="t=0")
    if flips:
        st = resync_oracle_from_gpu(st, g)
    log = []
    for t in range(1, gens + 1):
        prev_pf = g["pf"]
        for h in hs:
            h.step(problem, 1)
        st = O.pso_run(problem, N, D, lb, ub, seed=seed, n_gens=1, W=W, state=st)
        g = _sharded_pso_state(hs, D)
        flips = compare_pso(g, st, prev_pf_gpu=prev_pf, label=f"W={W} t={t}")
        if flips:
            log.append((t, flips))
            st = resync_oracle_from_gpu(st, g)
    assert len(log) <= 2, log


@pytest.mark.parametrize("W", [2, 4])
def test_pso_peer_tell_shard_tie_lowest_global_index(W):
    """S:349 / R-11 through the real exchange: the same minimum planted in EVERY shard (as
    caller fitness through ask/tell) must select the lowest global index, on every rank;
    a later generation whose minimum equals the incumbent gf must not move gbest."""
    N, D = 40, 6
    hs = _pso_group(W, N, D, -1, 1, 3)
    bounds = np.cumsum([0] + [ev.shard_rows(N, W, r)[1] for r in range(W)])
    X0 = []
    for r, h in enumerate(hs):
        Xa = h.ask()
        h.sync()
        X0.append(Xa.cpu().numpy()[:, :D].copy())
        f = torch.full((bounds[r + 1] - bounds[r],), 5.0, device="cuda")
        f[-1] = 1.0                      # the last row of every shard ties at the minimum
        h.tell(f)
    X0 = np.concatenate(X0)
    for h in hs:
        gf, gi, row = h.best()
        assert (gf, gi) == (1.0, bounds[1] - 1)
        assert np.array_equal(row, X0[bounds[1] - 1])
    for r, h in enumerate(hs):      # generation 1: the minimum equals the incumbent, elsewhere
        h.ask()
        f = torch.full((bounds[r + 1] - bounds[r],), 3.0, device="cuda")
        f[0] = 1.0
        h.tell(f)
    for h in hs:
        gf, gi, row = h.best()
        assert (gf, gi) == (1.0, bounds[1] - 1)          # strict: the incumbent stays
        assert np.array_equal(row, X0[bounds[1] - 1])
        assert list(h.history()) == [1.0, 1.0]


def _ipc_worker(rank, world, q_in, q_out, N, D, gens, problem, seed):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch as T
    import paper_2301_12457_b200 as EV
    T.cuda.set_device(0)
    lb, ub = EV.evox.DEFAULT_BOUNDS[problem]
    h = EV.PSO(N, D, lb, ub, seed=seed, rank=rank, world=world, peer_timeout_ms=60000)
    q_out.put((rank, h.mailbox_ipc()))
    handles = q_in.get()
    h.connect_ipc(handles)
    h.step(problem, gens)
    h.sync()
    q_out.put((rank, h.view("X").cpu().numpy()[:, :D].copy(), h.view("F").cpu().numpy().copy(),
               h.best(), h.history()))
    h.close()


@pytest.mark.parametrize("W", [2, 4, 8])
def test_pso_peer_ipc_processes_vs_oracle(W):
    """W processes on one GPU, mailboxes mapped through CUDA IPC (the multi-process form
    of the exchange): after the run, the population, the best and the history against
    oracle_pso_run(W)."""
    import torch.multiprocessing as mp
    N, D, gens, problem, seed = 120, 16, 12, "rastrigin", 3
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    q_in = [ctx.Queue() for _ in range(W)]
    procs = [ctx.Process(target=_ipc_worker, args=(r, W, q_in[r], q_out, N, D, gens, problem,
                                                   seed)) for r in range(W)]
    for p in procs:
        p.start()
    hd = dict(q_out.get(timeout=300) for _ in range(W))
    for r in range(W):
        q_in[r].put([hd[i] for i in range(W)])
    res = {}
    for _ in range(W):
        item = q_out.get(timeout=300)
        res[item[0]] = item[1:]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    lb, ub = WL.BOUNDS[problem]
    st = O.pso_run(problem, N, D, lb, ub, seed=seed, n_gens=gens, W=W)
    X = np.concatenate([res[r][0] for r in range(W)])
    F = np.concatenate([res[r][1] for r in range(W)])
    if not np.array_equal(X, st.X):  # only a near-tie decision may explain a difference
        assert_positions(X, st.X, "IPC X")
    assert_fitness(F, O.evaluate(problem, X), "IPC f")
    for r in range(W):
        gf, gi, row = res[r][2]
        assert gi == st.gidx or near_tie(gf, st.gf)
        assert_fitness(np.array([gf]), np.array([float(st.gf)]), "IPC gf")
        assert_fitness(res[r][3], np.asarray(st.hist, np.float64), "IPC hist")


# ------------------------------------------------------------------ CSO
def _cso_group(W, N, D, lb, ub, B, seed, phi=0.0):
    hs = [ev.CSO(N, D, lb, ub, phi=phi, block=B, seed=seed, rank=r, world=W,
                 stream=torch.cuda.Stream()) for r in range(W)]
    bases = [h.state_base() for h in hs]
    for h in hs:
        h.connect_local(bases)
    return hs


def cso_flipped_pairs_are_near_ties(Xg, Xo, f_prev, N, B, t, seed):
    """Rows that differ after a CSO generation must belong to pairs whose winner decision
    flipped -- allowed only at a near-tie of the pre-generation fitness (R-9)."""
    rows = np.nonzero((Xg != Xo).any(1))[0]
    for r in rows:
        blk = int(r) // B
        Bb = min(B, N - blk * B)
        loc = int(r) - blk * B
        partner = None
        for a, b in O.cso_pairs(Bb, blk, t, seed):
            if a == loc:
                partner = blk * B + int(b)
            elif b == loc:
                partner = blk * B + int(a)
        assert partner is not None, f"row {r} is unpaired but changed"
        assert near_tie(f_prev[r], f_prev[partner]), (t, int(r), partner, f_prev[r],
                                                      f_prev[partner])
    return rows.size


def cso_oracle_parity(step, gpu_state, problem, N, D, B, seed, gens, phi=0.0):
    """Step a CSO (single handle or sharded group) and the oracle side by side."""
    lb, ub = WL.BOUNDS[problem]
    X, V, f, F64 = O.cso_init(problem, N, D, lb, ub, seed)
    step(0)
    Xg, Vg, fg, hist = gpu_state()
    assert np.array_equal(Xg, X)
    assert_fitness(fg, F64, "CSO t=0 f")
    f = fg.copy()  # decisions use the GPU's fp32 fitness (R-9)
    resync = 0
    for t in range(gens):
        f_prev = f.copy()
        step(1)
        O.cso_generation(problem, X, V, f, F64, B, t, seed, lb, ub, phi=phi)
        Xg, Vg, fg, hist = gpu_state()
        if not np.array_equal(Xg, X):
            cso_flipped_pairs_are_near_ties(Xg, X, f_prev, N, B, t, seed)
            resync += 1
            X, V = Xg.copy(), Vg.copy()
        else:
            assert np.array_equal(Vg, V)
        assert_fitness(fg, O.evaluate(problem, Xg), f"CSO t={t + 1} f")
        f = fg.copy()
        F64 = O.evaluate(problem, X)
        assert len(hist) == t + 2 and hist[-1] == f.min()
    assert (np.diff(hist) <= 0).all()  # the best individual always wins its pair
    return resync


@pytest.mark.parametrize("W,N,D,B,problem,phi", [(2, 64, 33, 64, "rastrigin", 0.0),
                                                 (3, 50, 100, 50, "ackley", 0.0),
                                                 (4, 96, 300, 30, "sphere", 0.0),
                                                 (8, 203, 20, 203, "griewank", 0.0),
                                                 (4, 256, 40, 64, "ackley", 0.2),
                                                 (8, 203, 57, 203, "rastrigin", 0.1)])
def test_cso_sharded_vs_oracle(W, N, D, B, problem, phi):
    """Pairs straddling shards (B up to pop: global pairing) and phi != 0 (x-bar from
    exchanged fixed-point column sums, R-15) against oracle_cso_generation."""
    lb, ub = WL.BOUNDS[problem]
    hs = _cso_group(W, N, D, lb, ub, B, 4, phi=phi)

    def step(n):
        for h in hs:
            h.step(problem, n)
        for h in hs:
            h.sync()

    def state():
        cat = lambda k: np.concatenate([h.view(k).cpu().numpy() for h in hs])  # noqa: E731
        hist = hs[0].history()
        for h in hs[1:]:
            assert np.array_equal(h.history(), hist)
        return cat("X")[:, :D], cat("V")[:, :D], cat("F"), hist

    resync = cso_oracle_parity(step, state, problem, N, D, B, 4, gens=15, phi=phi)
    assert resync <= 2


def test_cso_planted_ties_lower_global_index_wins():
    """R-8 on the GPU, single handle and 4 shards with straddling pairs: every row is a sign
    pattern of one vector (Sphere ties exactly, on both sides), so every pair is a tie and
    the LOWER global index must win (pass unchanged) -- the same rows as the oracle's."""
    N, D, B, seed = 64, 12, 64, 9
    rng = np.random.default_rng(1)
    a = rng.uniform(0.5, 2.0, D).astype(np.float32)
    X0 = (a * rng.choice([-1.0, 1.0], (N, D))).astype(np.float32)
    Xo, Vo = X0.copy(), np.zeros_like(X0)
    F64 = O.evaluate("sphere", Xo)
    fo = F64.astype(np.float32)
    O.cso_generation("sphere", Xo, Vo, fo, F64, B, 0, seed, -5.12, 5.12)
    for W in (1, 4):
        hs = [ev.CSO(N, D, -5.12, 5.12, block=B, seed=seed, rank=r, world=W,
                     stream=torch.cuda.Stream()) for r in range(W)]
        if W > 1:
            bases = [h.state_base() for h in hs]
            for h in hs:
                h.connect_local(bases)
        for r, h in enumerate(hs):  # plant the population before generation 0's evaluation
            r0, n = ev.shard_rows(N, W, r)
            h.view("X")[:, :D].copy_(torch.from_numpy(X0[r0:r0 + n]))
        torch.cuda.synchronize()
        for h in hs:
            h.step("sphere", 0)
        f0 = np.concatenate([h.view("F").cpu().numpy() for h in hs])
        assert (f0 == f0[0]).all()
        for h in hs:
            h.step("sphere", 1)
        for h in hs:
            h.sync()
        Xg = np.concatenate([h.view("X").cpu().numpy()[:, :D] for h in hs])
        assert np.array_equal(Xg, Xo), W
        for p, q in O.cso_pairs(B, 0, 0, seed):
            assert np.array_equal(Xg[min(p, q)], X0[min(p, q)])


# ------------------------------------------------------------------ DE
def _de_group(W, N, D, lb, ub, seed):
    hs = [ev.DE(N, D, lb, ub, seed=seed, rank=r, world=W, stream=torch.cuda.Stream())
          for r in range(W)]
    bases = [h.state_base() for h in hs]
    for h in hs:
        h.connect_local(bases)
    return hs


@pytest.mark.parametrize("W,N,D,problem", [(2, 64, 37, "ackley"), (3, 50, 100, "sphere"),
                                           (4, 97, 300, "rastrigin"), (8, 203, 20, "griewank")])
def test_de_sharded_vs_oracle(W, N, D, problem):
    """Donors drawn from the whole population and read across shards through peer memory,
    against oracle_de_generation, every generation (view() gathers without touching the
    state the peers read)."""
    lb, ub = WL.BOUNDS[problem]
    seed, gens = 6, 15
    hs = _de_group(W, N, D, lb, ub, seed)
    for h in hs:
        h.step(problem, 0)
    X, f, F64 = O.de_init(problem, N, D, lb, ub, seed)
    for h in hs:
        h.sync()
    Xg = np.concatenate([h.view("X").cpu().numpy()[:, :D] for h in hs])
    assert np.array_equal(Xg, X)
    f = np.concatenate([h.view("F").cpu().numpy() for h in hs])
    resync = 0
    for t in range(gens):
        X0 = X.copy()
        for h in hs:
            h.step(problem, 1)
        for h in hs:
            h.sync()
        O.de_generation(problem, X, f, F64, t, seed, lb, ub)
        Xg = np.concatenate([h.view("X").cpu().numpy()[:, :D] for h in hs])
        fg = np.concatenate([h.view("F").cpu().numpy() for h in hs])
        diff = np.nonzero((Xg != X).any(1))[0]
        for i in diff:
            r = O.de_indices(N, int(i), t, seed)
            U = O.draw(1, D, int(i), t, 10, seed)[0]
            u = O.de_trial_with(X0[i], X0[r[0]], X0[r[1]], X0[r[2]], U,
                                O.de_jrand(D, int(i), t, seed), 0.5, 0.9, lb, ub)
            assert near_tie(float(O.evaluate(problem, u[None])[0]),
                            float(O.evaluate(problem, X0[i][None])[0])), (t, int(i))
        if diff.size:
            resync += 1
            X = Xg.copy()
        assert_fitness(fg, O.evaluate(problem, Xg), f"DE W={W} t={t + 1} f")
        f = fg.copy()
        F64 = O.evaluate(problem, X)
        hist = hs[0].history()
        assert hist[-1] == f.min()
    assert resync <= 2
