import time, sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2301_12457_b200 as ev
torch.cuda.set_device(0)
for cfg in [("griewank", 1_000_000, 100), ("ackley", 1_000_000, 1000), ("griewank", 1_000_000, 100), ("rosenbrock", 1_000_000, 100)]:
    p, N, D = cfg
    for rep in range(2):
        t0 = time.perf_counter()
        h = ev.PSO(N, D, -5, 5, seed=0)
        t1 = time.perf_counter()
        h.sync()
        t2 = time.perf_counter()
        h.step(p, 0)
        h.sync()
        t3 = time.perf_counter()
        h.step(p, 1)
        h.sync()
        t4 = time.perf_counter()
        h.close()
        t5 = time.perf_counter()
        print(p, N, D, rep, f"init {1e3*(t1-t0):.1f} sync {1e3*(t2-t1):.1f} gen0 {1e3*(t3-t2):.1f} step1 {1e3*(t4-t3):.1f} close {1e3*(t5-t4):.1f} ms", flush=True)
