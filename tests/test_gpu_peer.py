"""The in-kernel peer-memory winner exchange on ONE GPU.

W ranks are W handles of one process (each on its own stream, mailboxes
connected by pointer) or W processes (mailboxes connected by CUDA IPC).  The
sharded trajectory must equal the single-shard one bitwise (R-11)."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2301_12457_b200 as ev  # noqa: E402
from paper_2301_12457_b200 import evox as E  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


def _group(W, N, D, lb, ub, seed, **kw):
    hs = [ev.PSO(N, D, lb, ub, seed=seed, rank=r, world=W, stream=torch.cuda.Stream(), **kw)
          for r in range(W)]
    boxes = [h.mailbox()[0] for h in hs]
    for h in hs:
        h.connect_local(boxes)
    return hs


def _concat(hs, field, D):
    return np.concatenate([h.view(field).cpu().numpy()[:, :D] if field in "XVP"
                           else h.view(field).cpu().numpy() for h in hs])


@pytest.mark.parametrize("W,N,D,problem", [(2, 64, 37, "ackley"), (3, 50, 100, "rosenbrock"),
                                           (4, 97, 1000, "rastrigin"), (8, 203, 20, "griewank"),
                                           (2, 9, 4099, "sphere")])
def test_peer_group_equals_single_shard(W, N, D, problem):
    lb, ub = {"ackley": (-32.768, 32.768), "rosenbrock": (-5, 10), "rastrigin": (-5.12, 5.12),
              "griewank": (-600, 600), "sphere": (-5.12, 5.12)}[problem]
    ref = ev.PSO(N, D, lb, ub, seed=5)
    ref.step(problem, 0)
    ref.step(problem, 40)
    hs = _group(W, N, D, lb, ub, 5)
    for h in hs:          # generation 0 (evaluate X0 + tell + exchange): all ranks in flight
        h.step(problem, 0)
    for _ in range(2):    # 40 generations as two graph-replayed chunks per rank
        for h in hs:
            h.step(problem, 20)
    for h in hs:
        h.sync()
    for k in ("X", "V", "P"):
        assert np.array_equal(_concat(hs, k, D), ref.view(k).cpu().numpy()[:, :D]), k
    for k in ("F", "PF"):
        assert np.array_equal(_concat(hs, k, D), ref.view(k).cpu().numpy()), k
    rb = ref.best()
    for h in hs:
        b = h.best()
        assert b[0] == rb[0] and b[1] == rb[1] and np.array_equal(b[2], rb[2])
        assert np.array_equal(h.history(), ref.history())


def test_peer_group_ask_tell():
    W, N, D, p = 3, 31, 12, "ackley"
    ref = ev.PSO(N, D, -32.768, 32.768, seed=8)
    ref.step(p, 6)
    hs = _group(W, N, D, -32.768, 32.768, 8)
    for _ in range(7):
        for h in hs:
            X = h.ask()
            with torch.cuda.stream(h.stream):
                f = ev.evaluate(p, X, dim=D, stream=h.stream)
            h.tell(f)
    for h in hs:
        h.sync()
    assert np.array_equal(_concat(hs, "X", D), ref.view("X").cpu().numpy()[:, :D])
    assert hs[0].best()[:2] == ref.best()[:2]


def test_peer_timeout_reports_exchange_error():
    hs = _group(2, 16, 8, -1, 1, 1, peer_timeout_ms=1500)
    hs[0].step("sphere", 0)          # rank 1 never steps
    with pytest.raises(E.ExchangeError):
        hs[0].sync()
    with pytest.raises(E.PoisonedError):
        hs[0].step("sphere", 1)


def test_peer_connect_contract():
    h = ev.PSO(10, 4, -1, 1, seed=0, rank=0, world=2)
    with pytest.raises(E.ContractError):
        h.step("sphere", 1)      # world 2, neither NCCL nor connected
    g = ev.PSO(10, 4, -1, 1, seed=0)
    g.step("sphere", 1)
    with pytest.raises(E.ContractError):
        g.connect_local([g.mailbox()[0]])   # connect after stepping


def _ipc_worker(rank, world, q_in, q_out, N, D, gens):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch as T
    import paper_2301_12457_b200 as EV
    T.cuda.set_device(0)
    h = EV.PSO(N, D, -5.12, 5.12, seed=3, rank=rank, world=world)
    q_out.put((rank, h.mailbox_ipc()))
    handles = q_in.get()
    h.connect_ipc(handles)
    h.step("rastrigin", gens)
    h.sync()
    q_out.put((rank, h.view("X").cpu().numpy()[:, :D].copy(), h.best(), h.history()))
    h.close()


def test_peer_ipc_two_processes_one_gpu():
    """Two processes on the same GPU, mailboxes mapped through CUDA IPC."""
    import torch.multiprocessing as mp
    N, D, gens, W = 40, 16, 6, 2
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    q_in = [ctx.Queue() for _ in range(W)]
    procs = [ctx.Process(target=_ipc_worker, args=(r, W, q_in[r], q_out, N, D, gens))
             for r in range(W)]
    for p in procs:
        p.start()
    hd = dict(q_out.get(timeout=180) for _ in range(W))
    for r in range(W):
        q_in[r].put([hd[i] for i in range(W)])
    res = {}
    for _ in range(W):
        item = q_out.get(timeout=300)
        res[item[0]] = item[1:]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    ref = ev.PSO(N, D, -5.12, 5.12, seed=3)
    ref.step("rastrigin", gens)
    X = np.concatenate([res[r][0] for r in range(W)])
    assert np.array_equal(X, ref.view("X").cpu().numpy()[:, :D])
    for r in range(W):
        assert res[r][1][:2] == ref.best()[:2]
        assert np.array_equal(res[r][2], ref.history())
