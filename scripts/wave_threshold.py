"""Wave / flat grid against the persistent grid-stride walk at few-wave populations (measurement
script for EVOX_WAVE_MIN_WAVES): per point, 20 generations timed with CUDA events on the handle's
stream, once as the library dispatches (flags 0) and once with EVOX_FLAG_NO_WAVE.
    EVOX_LIB=<variant .so> python scripts/wave_threshold.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2301_12457_b200 as ev  # noqa: E402
from paper_2301_12457_b200 import evox as E  # noqa: E402
from paper_2301_12457_b200 import workloads as WL  # noqa: E402

PEAK = 6537.6
POINTS = [("ackley", 10_000, 4096), ("ackley", 40_000, 4096), ("ackley", 20_000, 2048),
          ("ackley", 80_000, 2048), ("ackley", 12_000, 3000), ("ackley", 50_000, 1500),
          ("ackley", 34_000, 1000), ("ackley", 1_000_000, 1000), ("sphere", 340_000, 100),
          ("rosenbrock", 700_000, 100), ("ackley", 4_100, 8192), ("ackley", 2_000, 20_000),
          ("sphere", 150_000, 250)]
if len(sys.argv) > 1 and sys.argv[1] == "big":
    POINTS = [pt for pt in POINTS if pt[2] in (1000, 1500, 2048, 3000, 4096)]
torch.cuda.set_device(0)
for p, N, D in POINTS:
    res = []
    for flags in (0, E.FLAG_NO_WAVE):
        lb, ub = WL.BOUNDS[p]
        h = ev.PSO(N, D, lb, ub, seed=0, flags=flags)
        h.step(p, 4)
        h.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(h.stream)
        h.step(p, 20)
        e1.record(h.stream)
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        ld = (D + 3) // 4 * 4
        frac = (20.0 * N * ld + 10.0 * N) / (us * 1e-6) / 1e9 / PEAK
        res.append(f"{'dispatch' if flags == 0 else 'no_wave'} {us:8.1f} us {frac:.3f}")
        h.close()
    print(f"{p:10s} pop {N:7d} dim {D:6d}  " + "  |  ".join(res), flush=True)
