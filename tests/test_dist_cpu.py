"""World-size-2 (gloo, CPU) tests of the N>1 host logic: row sharding through the
C-ABI, the unique-id broadcast plumbing, and the per-generation winner-record
exchange protocol (the paper's all-gather of P:583-587) run on
oracle shards -- the trajectory must equal the single-process run bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ord(f):
    """Order-preserving f32 -> u32 (NaN -> +inf, -0 -> +0): the record key's high word."""
    f = np.float32(np.inf) if np.isnan(f) else np.float32(f)
    if f == 0:
        f = np.float32(0.0)
    b = int(np.array([f], np.float32).view(np.uint32)[0])
    return (~b) & 0xFFFFFFFF if b & 0x80000000 else b | 0x80000000


def _worker(rank, world, port, N, D, n_gens, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle as O
    import paper_2301_12457_b200 as ev

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # unique-id plumbing: rank 0's 128 bytes reach every rank
        buf = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            buf = torch.from_numpy(np.frombuffer(os.urandom(128), np.uint8).copy())
        dist.broadcast(buf, 0)
        ids = [torch.zeros(128, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(ids, buf)
        assert all(torch.equal(ids[0], x) for x in ids)

        row0, rows = ev.shard_rows(N, world, rank)
        lb, ub, seed, prob = -32.768, 32.768, 17, "ackley"
        w, pp, pg = 0.6, 2.5, 0.8
        X, V = O.pso_init(rows, D, row0, lb, ub, seed)
        P = X.copy()
        pf = np.full(rows, np.inf, np.float32)
        G = np.zeros(D, np.float32)
        gf, gidx = np.float32(np.inf), -1
        hist = []
        for t in range(n_gens + 1):
            if t > 0:
                O.pso_move(X, V, P, G, row0, t - 1, seed, w, pp, pg, lb, ub)
            f = O.evaluate(prob, X).astype(np.float32)
            O.pso_tell_rows(X, f, P, pf)
            # local winner record {key, row}
            i, m = O.argmin(f)
            key = (_ord(m) << 32) | (row0 + i)
            rec = torch.from_numpy(np.concatenate([[np.float64(0)], X[i].astype(np.float64)]))
            keys = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
            recs = [torch.zeros(D + 1, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(keys, torch.tensor([key - (1 << 63)], dtype=torch.int64))
            dist.all_gather(recs, rec)
            k = [int(x.item()) + (1 << 63) for x in keys]
            win = int(np.argmin(k))
            hi = k[win] >> 32
            bits = (hi & 0x7FFFFFFF) if hi & 0x80000000 else (~hi) & 0xFFFFFFFF
            fm = np.array([bits], np.uint32).view(np.float32)[0]
            hist.append(float(fm))
            if fm < gf:  # strict improvement (R-5)
                gf, gidx = fm, k[win] & 0xFFFFFFFF
                G = recs[win].numpy()[1:].astype(np.float32)
        out[rank] = (row0, X, V, P, pf, G, float(gf), int(gidx), hist)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,D,world", [(37, 9, 2), (64, 33, 2)])
def test_sharded_exchange_matches_single_process(N, D, world):
    import oracle as O
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, D, 12, out))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    ref = O.pso_run("ackley", N, D, -32.768, 32.768, seed=17, n_gens=12)
    X = np.concatenate([out[r][1] for r in range(world)])
    V = np.concatenate([out[r][2] for r in range(world)])
    P = np.concatenate([out[r][3] for r in range(world)])
    assert np.array_equal(X, ref.X) and np.array_equal(V, ref.V) and np.array_equal(P, ref.P)
    for r in range(world):
        assert np.array_equal(out[r][5], ref.G)
        assert out[r][6] == ref.gf and out[r][7] == ref.gidx
        assert out[r][8] == ref.hist
