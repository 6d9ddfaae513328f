"""bench.py's N>1 flow (torchrun, one rank per process, states / mailboxes mapped through CUDA
IPC, barrier + max over ranks) run with both ranks on cuda:0 (EVOX_BENCH_SAME_GPU=1, gloo
group): the JSON line contract for PSO (in-kernel peer exchange), CSO (IPC-connected shards)
and DE (cross-shard donors).  Timings of this mode are meaningless; the flow is what is tested."""
import json
import os
import random
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config,pop", [("H", 20000), ("C3", 20000), ("D1", 20000), ("C5", 400)])
def test_bench_two_ranks_same_gpu(config, pop):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    env = dict(os.environ, EVOX_BENCH_SAME_GPU="1")
    nproc = 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + random.randrange(300)),
           "bench.py", "--gpus", str(nproc), "--config", config, "--pop", str(pop), "--steps", "3",
           "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == nproc and d["steps"] == 3 and d["value"] > 0
    assert d["roofline"]["bound"] == "hbm" and d["gpu_launches"] >= 3
    assert d["config"]["pop"] == pop
    if config in ("H", "C5"):  # the key-first peer exchange kernel runs once per generation
        assert d["exchange"]["kernel"] == "k_pso_fin" and d["exchange"]["ms_per_gen"] > 0
        assert d["gpu_launches"] >= 6


@pytest.mark.parametrize("config", ["EH-rosenbrock", "E5-griewank"])
def test_bench_eval_line(config):
    """SURVEY §8(d) evox_eval bench line: one JSON line, roofline against HBM, an e2e number
    measured with host buffers (H2D of X and D2H of the fitness every step)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    cmd = [sys.executable, "bench.py", "--config", config, "--pop", "64", "--steps", "3",
           "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "2"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["unit"] == "populations evaluated/s" and d["value"] > 0 and d["gpu_launches"] == 3
    assert d["roofline"]["bound"] == "hbm" and d["roofline"]["frac"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 4 * 64 * ((d["config"]["dim"] + 3) // 4 * 4)
    assert d["e2e"]["d2h_bytes_per_step"] == 4 * 64
