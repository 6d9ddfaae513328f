"""Generation time along a trajectory (does the per-generation cost drift as the swarm converges?):
20-generation windows timed with CUDA events on the handle's stream, one config.
    python scripts/gen_drift.py H 300"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2301_12457_b200 as ev  # noqa: E402
from paper_2301_12457_b200 import workloads as WL  # noqa: E402

import pynvml  # noqa: E402

pynvml.nvmlInit()
nv = pynvml.nvmlDeviceGetHandleByIndex(0)


def nvml_line():
    sm = pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM)
    mem = pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_MEM)
    pw = pynvml.nvmlDeviceGetPowerUsage(nv) / 1000.0
    tmp = pynvml.nvmlDeviceGetTemperature(nv, pynvml.NVML_TEMPERATURE_GPU)
    rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(nv)
    return f"sm {sm} MHz mem {mem} MHz {pw:.0f} W {tmp} C reasons 0x{rs:x}"


cfg = WL.CONFIGS[sys.argv[1]]
total = int(sys.argv[2]) if len(sys.argv) > 2 else 200
torch.cuda.set_device(0)
lb, ub = WL.BOUNDS[cfg.problem]
h = ev.PSO(cfg.pop, cfg.dim, lb, ub, seed=0)
h.step(cfg.problem, 0)
done = 0
while done < total:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(h.stream)
    h.step(cfg.problem, 20)
    e1.record(h.stream)
    line = nvml_line() if False else None
    e1.synchronize()
    print(f"gens {done + 1:5d}-{done + 20:5d}: {e0.elapsed_time(e1) / 20 * 1e3:8.1f} us/gen  "
          f"gbest {h.best(with_row=False)[0]:.4g}  {nvml_line()}", flush=True)
    done += 20
