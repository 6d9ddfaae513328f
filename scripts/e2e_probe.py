"""Per-step host timing of the e2e loop (step(1) + synchronising best()) for one config, to see
whether the e2e overhead over the device time is per step or one-off.
    python scripts/e2e_probe.py H 100"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_12457_b200 as ev  # noqa: E402
from paper_2301_12457_b200 import workloads as WL  # noqa: E402

cfg = WL.CONFIGS[sys.argv[1]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100
torch.cuda.set_device(0)
lb, ub = WL.BOUNDS[cfg.problem]
flags = ev.evox.FLAG_NO_GRAPH if (len(sys.argv) > 3 and sys.argv[3] == "nograph") else 0
h = ev.PSO(cfg.pop, cfg.dim, lb, ub, seed=0, flags=flags)
print("flags", flags)
h.step(cfg.problem, 0)
h.sync()
for mode in ("step1+best", "step1+sync", "step1 x n then sync", "stepN"):
    ts = []
    t0 = time.perf_counter()
    if mode == "stepN":
        h.step(cfg.problem, n)
        h.sync()
    else:
        for _ in range(n):
            a = time.perf_counter()
            h.step(cfg.problem, 1)
            if mode == "step1+best":
                h.best(with_row=True)
            elif mode == "step1+sync":
                h.sync()
            ts.append(time.perf_counter() - a)
        h.sync()
    tot = time.perf_counter() - t0
    ts = np.array(ts) * 1e3 if ts else np.array([0.0])
    print(f"{mode:22s} total {tot * 1e3:9.2f} ms  per step {tot * 1e3 / n:8.3f} ms  "
          f"first {ts[0]:8.3f}  median {np.median(ts):8.3f}  max {ts.max():8.3f}", flush=True)
