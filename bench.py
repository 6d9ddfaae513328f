#!/usr/bin/env python
"""Benchmark of the EvoX PSO/CSO generation on B200 (BASELINE.json metric).

A "step" is one generation of the whole hot path (Philox r1/r2,
velocity/position update + clip, fitness, pbest, gbest argmin, and for N>1
the per-generation winner exchange) over the whole population.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config H|C1|C2|C3|C4g|C4r|C5]
                    [--impl ours|reference] [--no-cpu-baseline]

N>1 is launched with torchrun (one rank per GPU, NCCL): the population is
row-sharded across ranks (strong scaling: fixed N_pop), one NCCL all-gather of
the W winner records per generation.  Rank 0 prints ONE JSON line.

--impl reference times the CPU oracle (the only reference this tier has) on a
bounded row sample of the same workload, on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2301_12457_b200 import workloads as WL  # noqa: E402

METRIC = "generations/s and individual-dims/s at 1/2/4/8 B200; % HBM roofline"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def gen_kernel_name(cfg, rows, world):
    """The generation kernel evox_*_step launches for this shard (mirrors the C-ABI's
    dispatch: single-CTA persistent <= 2^14 elements, cooperative persistent <= 2^25 for
    PSO at W = 1, beyond 2^25 elements the flat-tile kernel for PSO rows of <= 256 floats and
    the wave grid for rows of > 256 floats (Griewank: > 4096), else one
    k_*_gen launch per generation)."""
    ld = (cfg.dim + 3) // 4 * 4
    n = rows * ld
    if cfg.algo == "pso" and world == 1 and n <= 16384:
        return f"k_pso_run_small<{cfg.problem}>"
    if cfg.algo == "pso" and world == 1 and n <= (1 << 25):
        return f"k_pso_run_mid<{cfg.problem}>"
    if cfg.algo == "pso" and n > (1 << 25) and ld <= 256:
        return f"k_pso_gen_flat<{cfg.problem}>"
    if cfg.algo == "pso" and n > (1 << 25) and (ld > 4096 or (
            ld > 256 and cfg.problem != "griewank" and (rows + 7) // 8 >= 3 * 148 * 4)):
        return f"k_pso_gen_wave<{cfg.problem}>"
    if cfg.algo == "de" and ld <= 256:
        return f"k_de_gen_flat<{cfg.problem}>"
    return f"k_{cfg.algo}_gen<{cfg.problem}>"


NOMINAL_HBM_GBS = 8000.0  # B200 nominal (DGX figure; 7.7 TB/s HGX), context for "frac"


def config_dict(cfg, world, exchange):
    """The `config` of the JSON line -- identical in the GPU arm and the reference arm."""
    par = f"row-sharded x{world}"
    if world > 1:
        kind = {"pso": "peer-memory key-first (in-kernel)" if exchange == "peer" else "nccl",
                "cso": "peer-memory pairs" if exchange == "peer" else "nccl",
                "de": "peer-memory donors", "eval": "none (independent rows)"}[cfg.algo]
        par += f", exchange={kind}"
    if cfg.algo == "eval":
        l2 = "X (4 GB) > L2: inputs larger than L2, no flush needed"
    else:
        l2 = ("state (X,V,P) > L2: inputs larger than L2, no flush needed"
              if 12 * cfg.pop * cfg.dim > 2 * 126e6 else "state comparable to L2")
    return {"workload": cfg.note, "algo": cfg.algo, "problem": cfg.problem, "pop": cfg.pop,
            "dim": cfg.dim, "seed": 1000 if cfg.algo == "eval" else 0, "parallelism": par,
            "l2": l2}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            v = float(json.load(fh)["hbm_gbs"])
        return v, "measured (MEASURED_PEAKS.json hbm_gbs: copy, read+write bytes)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def algorithmic_bytes(cfg, rows):
    """Bytes one generation must move; DESIGN.md §5 states them.

    PSO: per element X r+w (8), V r+w (8), P read-or-write (4) = 20 B; per row
    imp r+w (2), pf read (4), f write (4) = 10 B (the rare pf write is not counted).
    CSO: per loser element Xl r+w, Vl r+w, Xw read = 20 B, i.e. 10 B per population
    element; per pair f reads (8) + loser f write (4) = 6 B per row.
    DE: per element the target and three donor rows read (16) + the trial written (4).
    eval: X read (4 B/element) + f written (4 B/row)."""
    D = cfg.dim
    if cfg.algo == "eval":  # Problem.evaluate: read X (4 B/element), write f (4 B/row)
        return 4 * D * rows + 4 * rows
    if cfg.algo == "pso":
        return 20 * D * rows + 10 * rows
    if cfg.algo == "de":  # target 4 + three donors 12 + trial write 4; sel 4+1, f 4+4 per row
        return 20 * D * rows + 13 * rows
    return 10 * D * rows + 6 * rows


class ClockSampler:
    """SM clock, power and clock-event (throttle) reasons sampled DURING the timed region:
    NVML every 2 ms plus one sample at start and one at stop (so even a sub-millisecond
    region is bracketed); nvidia-smi polling as a fallback."""
    BITS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
            0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, power_w, reasons bitmask)
        self.stop_ev = threading.Event()
        self.th = None
        self.nvml = None

    def _sample(self):
        n, h = self.nvml, self.h
        try:
            rs = n.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            rs = n.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.rows.append((n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM),
                          n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM),
                          n.nvmlDeviceGetPowerUsage(h) / 1000.0, int(rs)))

    def _loop(self):
        while not self.stop_ev.wait(0.002):
            self._sample()

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._sample()
        except Exception:
            self.nvml = None
            return
        self.th = threading.Thread(target=self._loop, daemon=True)
        self.th.start()

    def stop(self):
        if self.nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        self.stop_ev.set()
        self.th.join(timeout=2)
        self._sample()
        sm = [r[0] for r in self.rows]
        reasons = sorted({name for r in self.rows for bit, name in self.BITS.items() if r[3] & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "power_w_max": max(r[2] for r in self.rows),
                "samples": len(self.rows), "source": "nvml, 2 ms + bracketing samples"}


def ncu_traffic(cfg_name):
    """DRAM bytes per launch of the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        v = d.get(cfg_name, {}).get("dram_bytes_per_launch")
        return float(v) if v is not None else None
    except Exception:
        return None


def cpu_baseline(cfg, target_s=12.0):
    """The oracle as it stands, on the host cores, over a bounded row sample of the workload
    (2 generations: move + evaluate + tell), extrapolated to whole-population gens/s; the same
    measured single-threaded on a smaller sample (nproc, CPU model, threads)."""
    cores = os.cpu_count() or 1
    D = cfg.dim
    rows = _sample_rows(cfg, cores, target_s / 2)
    gen = _oracle_gen(cfg, rows, cores)
    t0 = time.perf_counter()
    for t in range(2):
        gen(t)
    t_gen = (time.perf_counter() - t0) / 2
    frac = rows / cfg.pop
    gens_per_s = frac / t_gen
    rows1 = max(4, min(rows, _sample_rows(cfg, 1, 1.5)))
    gen1 = _oracle_gen(cfg, rows1, 1)
    t0 = time.perf_counter()
    gen1(0)
    t1 = time.perf_counter() - t0
    what = "2 evaluations" if cfg.algo == "eval" else "2 generations (move+eval+tell)"
    return {"value": gens_per_s, "unit": _unit(cfg), "cores": cores, "kind": "oracle",
            "sample": f"{rows} of {cfg.pop} rows x dim {D}, {what}, "
                      f"{t_gen * 2:.2f} s on {cores} threads; extrapolated linearly in rows",
            "individual_dims_per_s": gens_per_s * cfg.pop * D * (0.5 if cfg.algo == "cso" else 1),
            "cpu_model": cpu_model(), "nproc": cores,
            "single_thread": {"value": (rows1 / cfg.pop) / t1, "unit": _unit(cfg),
                              "sample": f"{rows1} rows, 1 generation, {t1:.2f} s"}}


def _device_info(dev):
    """device name, SM count, L2 size of the measuring GPU."""
    import torch
    p = torch.cuda.get_device_properties(dev)
    return {"name": p.name, "sms": p.multi_processor_count,
            "l2_mb": round(getattr(p, "L2_cache_size", 0) / 2**20, 1),
            "hbm_gb": round(p.total_memory / 1e9, 1)}


def _unit(cfg):
    return "populations evaluated/s" if cfg.algo == "eval" else "generations/s"


def run_eval(args, cfg, world, rank, local):
    """SURVEY §8(d) `evox_eval` line: one step = Problem.evaluate (Eq. (2)) of the whole
    population through the C-ABI -- this rank's contiguous row shard at N > 1 (rows are
    independent: no collective, weak in nothing but the shard).  X ~ U[lb, ub] (seeded torch
    generator: plumbing, not the method), padding columns 0, resident in HBM."""
    import torch
    import torch.distributed as dist

    import paper_2301_12457_b200 as ev
    torch.cuda.set_device(local)
    launched = "WORLD_SIZE" in os.environ
    if launched:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if launched:
            dist.barrier()
        torch.cuda.synchronize()

    row0, rows = ev.shard_rows(cfg.pop, world, rank)
    D, ld = cfg.dim, WL.round4(cfg.dim)
    lb, ub = WL.BOUNDS[cfg.problem]
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1000 + rank)
    X = torch.zeros((rows, ld), dtype=torch.float32, device="cuda")
    X[:, :D].uniform_(lb, ub, generator=gen)
    f = torch.empty(rows, dtype=torch.float32, device="cuda")
    stream = torch.cuda.Stream()
    for _ in range(args.warmup):
        ev.evaluate(cfg.problem, X, dim=D, out=f, stream=stream)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    evs[0].record(stream)
    for k in range(args.steps):
        ev.evaluate(cfg.problem, X, dim=D, out=f, stream=stream)
        evs[k + 1].record(stream)
    stream.synchronize()
    barrier()
    clk = clocks.stop()
    per = [evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)]
    t = torch.tensor([sum(per), sum(per) / len(per)], dtype=torch.float64, device="cuda")
    if launched:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t[0]) / args.steps
    k_avg_ms = float(t[1])

    # e2e through the C-ABI with host buffers: pinned host X -> device, evaluate, fitness -> host
    Xh = X.cpu().pin_memory()
    fh = torch.empty(rows, dtype=torch.float32).pin_memory()
    n_e2e = max(1, min(args.e2e_steps, 5))
    barrier()
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        with torch.cuda.stream(stream):
            X.copy_(Xh, non_blocking=True)
            ev.evaluate(cfg.problem, X, dim=D, out=f, stream=stream)
            fh.copy_(f, non_blocking=True)
        stream.synchronize()
    e2e = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    if launched:
        dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e[0])

    if rank == 0:
        peak, peak_src = hbm_peak()
        bytes_launch = algorithmic_bytes(cfg, rows)
        achieved = bytes_launch / (k_avg_ms * 1e-3) / 1e9
        value = 1e3 / ms_per_step
        line = {
            "metric": METRIC, "value": value, "unit": _unit(cfg), "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": config_dict(cfg, world, args.exchange),
            "individual_dims_per_s": value * cfg.pop * cfg.dim,
            "bytes_per_generation": algorithmic_bytes(cfg, cfg.pop),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "frac_of_nominal_8tbs": achieved / NOMINAL_HBM_GBS,
                         "traffic": ncu_traffic(args.config),
                         "kernel": f"k_eval<{cfg.problem}>", "kernel_ms": k_avg_ms,
                         "bytes_per_launch": bytes_launch, "peak_source": peak_src},
            "clocks": clk,
            "device": _device_info(local),
            "gpu_launches": args.steps,
            "e2e": {"value": n_e2e / e2e_s, "unit": _unit(cfg),
                    "h2d_bytes_per_step": 4 * cfg.pop * ld, "d2h_bytes_per_step": 4 * cfg.pop,
                    "steps": n_e2e,
                    "note": "per step: pinned host X -> device, evox_eval through the C-ABI, "
                            "fitness -> pinned host, stream sync"},
        }
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(line), flush=True)
    if launched:
        dist.destroy_process_group()


def _oracle_gen(cfg, rows, cores):
    """Initialise the oracle on `rows` rows of the workload; returns a callable that runs one
    generation (move + evaluate + tell) in place."""
    import oracle as O
    lb, ub = WL.BOUNDS[cfg.problem]
    D = cfg.dim
    if cfg.algo == "eval":
        X = WL.uniform_rows(rows, D, cfg.problem, seed=0)

        def gen(i):
            O.evaluate(cfg.problem, X, threads=cores)
    elif cfg.algo == "pso":
        box = [O.pso_run(cfg.problem, rows, D, lb, ub, seed=0, n_gens=0, threads=cores)]

        def gen(i):
            box[0] = O.pso_run(cfg.problem, rows, D, lb, ub, seed=0, n_gens=1, state=box[0],
                               threads=cores)
    elif cfg.algo == "de":
        X, f, F64 = O.de_init(cfg.problem, rows, D, lb, ub, 0, threads=cores)

        def gen(i):
            O.de_generation(cfg.problem, X, f, F64, i, 0, lb, ub, threads=cores)
    else:
        B = max(2, rows // 8 if rows % 16 == 0 else rows)
        X, V, f, F64 = O.cso_init(cfg.problem, rows, D, lb, ub, 0, threads=cores)

        def gen(i):
            O.cso_generation(cfg.problem, X, V, f, F64, B, i, 0, lb, ub, threads=cores)
    return gen


def _sample_rows(cfg, cores, seconds):
    """Rows of the workload one oracle generation covers in about `seconds` on `cores` threads,
    calibrated by timing one generation on a small sample (the oracle's speed varies by host)."""
    rows_c = int(max(4, min(cfg.pop, 2e5 / cfg.dim)))
    gen = _oracle_gen(cfg, rows_c, cores)
    t0 = time.perf_counter()
    gen(0)
    per_row = max((time.perf_counter() - t0) / rows_c, 1e-12)
    return int(max(4, min(cfg.pop, seconds / per_row)))


def run_reference(args, cfg, rank):
    """The reference arm: the CPU oracle, as it stands, timed per generation on a bounded row
    sample of the same workload (this tier has no installable reference implementation);
    the line's `config` is the GPU arm's, the sample is stated in cpu_baseline.sample."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    D = cfg.dim
    # whole run (sample init + warm-up + timed generations) within about two minutes
    rows = _sample_rows(cfg, cores, 90.0 / max(1, args.steps + args.warmup + 1))
    gen = _oracle_gen(cfg, rows, cores)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        gen(i)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    value = (rows / cfg.pop) / t
    sample = (f"{rows} of {cfg.pop} rows x dim {D} per step, oracle on {cores} host threads, "
              f"extrapolated linearly in rows")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": _unit(cfg),
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3 * cfg.pop / rows, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(cfg, args.gpus, args.exchange),
            "individual_dims_per_s": value * cfg.pop * D * (0.5 if cfg.algo == "cso" else 1),
            "cpu_baseline": {"value": value, "unit": _unit(cfg), "cores": cores,
                             "kind": "oracle", "sample": sample, "cpu_model": cpu_model(),
                             "nproc": cores},
            "e2e": {"value": value, "unit": _unit(cfg), "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="H", choices=sorted(WL.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--sustained-s", type=float, default=1.5,
                    help="seconds of untimed generations before the sustained window (0: skip)")
    ap.add_argument("--pop", type=int, default=0, help="override the population (profiling only)")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="PSO winner exchange for N>1: in-kernel over NVLink peer memory "
                         "(default) or NCCL all-gather + select kernel")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = WL.CONFIGS[args.config]
    if args.pop:
        import dataclasses
        cfg = dataclasses.replace(cfg, pop=args.pop, note=cfg.note + f" [pop override {args.pop}]")

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, cfg, rank)
    if cfg.algo == "eval":
        return run_eval(args, cfg, world, rank, local)

    import torch
    import torch.distributed as dist

    import paper_2301_12457_b200 as ev

    # EVOX_BENCH_SAME_GPU=1: every rank on cuda:0 with a gloo group -- validates the N>1 flow
    # (IPC mailboxes, barriers, max-over-ranks) on a 1-GPU box; its timings are meaningless.
    same_gpu = os.environ.get("EVOX_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    launched = "WORLD_SIZE" in os.environ  # under torchrun: use the process group even at N=1
    cdev = "cpu" if same_gpu else "cuda"   # device of the collective tensors
    if launched:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nid = None
    # N>1 exchanges: PSO winner records through in-kernel peer mailboxes (default) or NCCL;
    # CSO shards connected through IPC-mapped states (default) or NCCL; DE always IPC-mapped
    peer = world > 1 and cfg.algo == "pso" and args.exchange == "peer"
    cso_peer = world > 1 and cfg.algo == "cso" and args.exchange == "peer"
    if world > 1 and not peer and not cso_peer and cfg.algo != "de":
        buf = torch.zeros(128, dtype=torch.uint8, device=cdev)
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(ev.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        nid = bytes(buf.cpu().numpy().tobytes())

    def barrier():
        if launched:
            dist.barrier()
        torch.cuda.synchronize()

    lb, ub = WL.BOUNDS[cfg.problem]

    def open_handle():
        """Handle setup through the public API: init from host lb/ub (copied H2D by the
        C-ABI), X0 from the seed on the device, N>1 peer mapping."""
        if cfg.algo == "de":  # shards read donors across GPUs: map every rank's state (IPC)
            h = ev.DE(cfg.pop, cfg.dim, lb, ub, seed=0, rank=rank, world=world)
            if world > 1:
                mine = torch.frombuffer(bytearray(h.state_ipc()), dtype=torch.uint8).to(cdev)
                allh = [torch.zeros(64, dtype=torch.uint8, device=cdev) for _ in range(world)]
                dist.all_gather(allh, mine)
                h.connect_ipc([bytes(x.cpu().numpy().tobytes()) for x in allh])
                barrier()
        elif cfg.algo == "cso":  # N>1: shards connected through IPC-mapped states (peer barrier)
            h = ev.CSO(cfg.pop, cfg.dim, lb, ub, block=cfg.pop // 8 if cfg.pop % 16 == 0 else 0,
                       seed=0, rank=rank, world=world, nccl_id=nid)
            if cso_peer:
                mine = torch.frombuffer(bytearray(h.state_ipc()), dtype=torch.uint8).to(cdev)
                allh = [torch.zeros(64, dtype=torch.uint8, device=cdev) for _ in range(world)]
                dist.all_gather(allh, mine)
                h.connect_ipc([bytes(x.cpu().numpy().tobytes()) for x in allh])
                barrier()
        else:
            h = ev.PSO(cfg.pop, cfg.dim, lb, ub, seed=0, rank=rank, world=world, nccl_id=nid)
        if peer:  # mailboxes of all ranks mapped into every rank through CUDA IPC
            mine = torch.frombuffer(bytearray(h.mailbox_ipc()), dtype=torch.uint8).to(cdev)
            allh = [torch.zeros(64, dtype=torch.uint8, device=cdev) for _ in range(world)]
            dist.all_gather(allh, mine)
            h.connect_ipc([bytes(x.cpu().numpy().tobytes()) for x in allh])
            barrier()
        return h

    h = open_handle()
    rows = h.info()["rows"]
    stream = h.stream
    h.step(cfg.problem, 0)          # generation 0: evaluate X0 + tell
    h.step(cfg.problem, args.warmup)  # untimed warm-up generations (graph capture included)
    h.sync()

    # ---- timed region: K generations, device-timed with CUDA events on the handle's stream
    h.set_timing(True)               # events around every generation kernel (dominant kernel)
    h.kernel_time(reset=True)
    if cfg.algo == "pso":
        h.fin_time(reset=True)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h.step(cfg.problem, args.steps)
    e1.record(stream)
    h.sync()
    barrier()
    clk = clocks.stop()
    ms_local = e0.elapsed_time(e1)
    k_ms, k_n, k_launch = h.kernel_time(reset=True)
    fin_ms, fin_launch = h.fin_time(reset=True) if cfg.algo == "pso" else (0.0, 0)
    h.set_timing(False)
    # one launch of the persistent small-population kernel runs all the steps
    t = torch.tensor([ms_local, k_ms / max(k_n, 1), fin_ms / max(fin_launch, 1)],
                     dtype=torch.float64, device=cdev)
    if launched:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total, k_avg_ms, fin_avg_ms = float(t[0]), float(t[1]), float(t[2])
    ms_per_step = ms_total / args.steps

    # ---- end to end: one whole job through the public API with host buffers, timed by the
    # host clock (max over ranks): init from host lb/ub (H2D inside the C-ABI), X0 from the
    # seed, generation 0, then every step evox_*_step(1) + a synchronising best() D2H of the
    # step's result (fitness, global index, best row), and the per-generation history D2H.
    h.close()
    barrier()
    t0 = time.perf_counter()
    h = open_handle()
    h.step(cfg.problem, 0)
    h.sync()
    t_setup = time.perf_counter()
    t_best = 0.0
    for _ in range(args.e2e_steps):
        h.step(cfg.problem, 1)
        tb = time.perf_counter()
        best = h.best(with_row=True)  # synchronising: waits for the step, then D2H
        t_best += time.perf_counter() - tb
    t_steps = time.perf_counter()
    hist = h.history()
    e2e_s = time.perf_counter() - t0
    parts = [e2e_s, t_setup - t0, t_steps - t_setup, t_best, e2e_s - (t_steps - t0)]
    e2e = torch.tensor(parts, dtype=torch.float64, device=cdev)
    if launched:
        dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    e2e_s, setup_s, steps_s, best_s, hist_s = (float(v) for v in e2e)
    e2e_h2d = 2 * 4 * cfg.dim / args.e2e_steps            # lb, ub (per job, amortised)
    # ---- sustained (after the e2e job, on its handle, so the job is timed as before): the same
    # K generations again after ~--sustained-s seconds of back-to-back (untimed) generations, once
    # the board's power limit has set its steady SM clock: at H the 1000 W cap (sw_power_cap)
    # takes the SM clock from ~1.9 GHz to ~1.56 GHz within ~0.5 s (DESIGN.md §7,
    # profiles/r02_power_drift.txt).  Reported next to the headline window.
    sus = None
    if args.sustained_s > 0:
        burn = int(min(5000, max(20, args.sustained_s * 1e3 / max(ms_per_step, 1e-3))))
        h.step(cfg.problem, burn)
        h.sync()
        h.set_timing(True)
        h.kernel_time(reset=True)
        clocks2 = ClockSampler(local)
        clocks2.start()
        barrier()
        e0.record(h.stream)
        h.step(cfg.problem, args.steps)
        e1.record(h.stream)
        h.sync()
        barrier()
        clk2 = clocks2.stop()
        k2_ms, k2_n, _ = h.kernel_time(reset=True)
        h.set_timing(False)
        t2 = torch.tensor([e0.elapsed_time(e1), k2_ms / max(k2_n, 1)], dtype=torch.float64,
                          device=cdev)
        if launched:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        sus = {"burn_in_generations": burn, "ms_per_step": float(t2[0]) / args.steps,
               "kernel_ms": float(t2[1]), "clocks": clk2}

    e2e_d2h = (4 + 8 + 4 * cfg.dim) + 4 * len(hist) / args.e2e_steps

    if rank == 0:
        peak, peak_src = hbm_peak()
        bytes_launch = algorithmic_bytes(cfg, rows)
        achieved = bytes_launch / (k_avg_ms * 1e-3) / 1e9
        kname = gen_kernel_name(cfg, rows, world)
        # the committed ncu entry is per generation of the kernel that actually runs
        traffic = ncu_traffic(args.config)
        gens_per_s = 1e3 / ms_per_step
        evaluated = cfg.pop * cfg.dim * (0.5 if cfg.algo == "cso" else 1.0)
        line = {
            "metric": METRIC,
            "value": gens_per_s,
            "unit": "generations/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic",
            "config": config_dict(cfg, world, args.exchange),
            "individual_dims_per_s": gens_per_s * evaluated,
            "bytes_per_generation": algorithmic_bytes(cfg, cfg.pop),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "frac_of_nominal_8tbs": achieved / NOMINAL_HBM_GBS,
                         "traffic": traffic,
                         "kernel": kname,
                         "kernel_ms": k_avg_ms, "bytes_per_launch": bytes_launch,
                         "peak_source": peak_src},
            "clocks": clk,
            "device": _device_info(local),
            # generation kernels timed by the library, the gbest-publication / key-first
            # exchange kernel k_pso_fin when it runs (wave grid, W > 1 peer exchange), and the
            # gbest select per step of the NCCL exchange
            "gpu_launches": k_launch + fin_launch + (args.steps if (cfg.algo == "pso" and world > 1
                                                                    and not peer) else 0),
            "exchange": ({"kernel": "k_pso_fin", "ms_per_gen": fin_avg_ms,
                          "frac_of_step": fin_avg_ms / ms_per_step,
                          "what": ("key-first peer exchange (8-byte keys to every rank; the "
                                   "winner row pulled over NVLink on a strict improvement) + "
                                   "gbest publication" if peer else
                                   "gbest publication after the wave-grid generation kernel")}
                         if fin_launch else None),
            "sustained": ({"value": 1e3 / sus["ms_per_step"], "unit": "generations/s",
                           "ms_per_step": sus["ms_per_step"],
                           "frac": bytes_launch / (sus["kernel_ms"] * 1e-3) / 1e9 / peak,
                           "kernel_ms": sus["kernel_ms"],
                           "burn_in_generations": sus["burn_in_generations"],
                           "clocks": sus["clocks"],
                           "note": "the same --steps generations timed the same way after "
                                   "burn_in_generations untimed back-to-back generations, when "
                                   "the board power limit has settled the SM clock"}
                          if sus else None),
            "e2e": {"value": args.e2e_steps / e2e_s, "unit": "generations/s",
                    "h2d_bytes_per_step": e2e_h2d, "d2h_bytes_per_step": e2e_d2h,
                    "steps": args.e2e_steps,
                    "breakdown_ms": {"setup": setup_s * 1e3,
                                     "per_step": steps_s * 1e3 / args.e2e_steps,
                                     "per_step_best_call": best_s * 1e3 / args.e2e_steps,
                                     "history": hist_s * 1e3,
                                     "device_step": ms_per_step},
                    "note": "host clock over one whole job through the C-ABI: init from host "
                            "lb/ub (H2D; the population is the method's own Philox init from "
                            "the seed, R-3), generation 0, then per step evox_*_step(1) + "
                            "synchronising best() D2H (fitness, index, best row), and the "
                            "history D2H; job setup amortised over the steps"},
        }
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(line), flush=True)
    h.close()
    if launched:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
