"""SURVEY §8(d) sweep grids on one GPU (the paper's scaling experiments, PAPER.md:700-702
§VII-A1; log axes PAPER.md:733, Fig. 6; plateau PAPER.md:741-742):

  * population sweep at dim 100: pop in 2^10 .. 2^20 and 10^6 (Sphere -- the paper's function
    -- and the C4 functions Griewank, Rosenbrock);
  * dimension sweep at pop 10^4: dim in 2^7 .. 2^17 and 10^5 (Sphere, Ackley);
  * dimension sweep at pop 100 (the paper's own dim-sweep population; latency-bound).

Each point: a PSO handle through the public API, generation 0 + 3 warm-up generations, then
20 generations timed on the handle's stream with CUDA events (and the library's per-kernel
events for the roofline).  Writes profiles/r02_sweeps.jsonl and prints a table.

    python scripts/sweep.py [--steps 20] [--out profiles/r02_sweeps.jsonl]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2301_12457_b200 import workloads as WL  # noqa: E402


def point(ev, torch, problem, pop, dim, steps, warmup=3):
    lb, ub = WL.BOUNDS[problem]
    h = ev.PSO(pop, dim, lb, ub, seed=0)
    h.step(problem, 0)
    h.step(problem, warmup)
    h.sync()
    cfg = WL.Config("sweep", "pso", problem, pop, dim, 1, "")
    kname = bench.gen_kernel_name(cfg, pop, 1)
    # device time of the whole step sequence (graph replay / persistent launches)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = h.stream
    e0.record(stream)
    h.step(problem, steps)
    e1.record(stream)
    h.sync()
    ms = e0.elapsed_time(e1) / steps
    # the generation kernel alone (events around every launch)
    h.set_timing(True)
    h.kernel_time(reset=True)
    h.fin_time(reset=True)
    h.step(problem, steps)
    k_ms, k_n, _ = h.kernel_time(reset=True)
    f_ms, f_n = h.fin_time(reset=True)
    h.set_timing(False)
    h.close()
    k_avg = k_ms / max(k_n, 1) + (f_ms / max(f_n, 1) if f_n else 0.0)
    peak, _ = bench.hbm_peak()
    b = bench.algorithmic_bytes(cfg, pop)
    return {"problem": problem, "pop": pop, "dim": dim, "gens_per_s": 1e3 / ms,
            "ms_per_gen": ms, "individual_dims_per_s": 1e3 / ms * pop * dim,
            "bytes_per_gen": b, "kernel": kname, "kernel_ms": k_avg,
            "achieved_gbs": b / (k_avg * 1e-3) / 1e9, "frac": b / (k_avg * 1e-3) / 1e9 / peak,
            "frac_step": b / (ms * 1e-3) / 1e9 / peak}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sweeps.jsonl"))
    args = ap.parse_args()
    import torch
    import paper_2301_12457_b200 as ev
    torch.cuda.set_device(0)
    grid = []
    for p in ("sphere", "griewank", "rosenbrock"):
        for n in [2 ** k for k in range(10, 21)] + [10 ** 6]:
            grid.append(("pop-sweep dim 100", p, n, 100))
    for p in ("sphere", "ackley"):
        for d in [2 ** k for k in range(7, 18)] + [10 ** 5]:
            grid.append(("dim-sweep pop 1e4", p, 10 ** 4, d))
    for d in [2 ** k for k in range(7, 18)] + [10 ** 5]:
        grid.append(("dim-sweep pop 100", "sphere", 100, d))
    rows = []
    with open(args.out, "w") as fh:
        for sweep, p, n, d in grid:
            r = point(ev, torch, p, n, d, args.steps)
            r["sweep"] = sweep
            rows.append(r)
            fh.write(json.dumps(r) + "\n")
            fh.flush()
            print(f"{sweep:18s} {p:10s} pop {n:8d} dim {d:7d}  {r['gens_per_s']:12.1f} gen/s  "
                  f"{r['individual_dims_per_s']:.3e} ind-dims/s  kernel {r['kernel_ms'] * 1e3:9.1f} us"
                  f"  {r['frac']:.3f} of HBM peak ({r['kernel']})", flush=True)


if __name__ == "__main__":
    main()
