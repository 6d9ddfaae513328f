"""Small runs of every kernel family for compute-sanitizer (memcheck/racecheck/synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_12457_b200 as ev  # noqa: E402

torch.cuda.set_device(0)
for D in (10, 100, 1003, 4099):
    for p in ("sphere", "ackley", "rastrigin", "griewank", "rosenbrock"):
        pso = ev.PSO(37, D, -5, 5, seed=1)
        pso.step(p, 3)
        X = pso.ask()
        pso.tell(ev.evaluate(p, X, dim=D, stream=pso.stream))  # on the handle's stream
        pso.view("P")
        pso.best()
        cso = ev.CSO(40, D, -5, 5, block=10, seed=1)
        cso.step(p, 3)
        cso.best()
        de = ev.DE(24, D, -5, 5, seed=1)
        de.step(p, 3)
        de.view("X")
        de.best()
pso = ev.PSO(300, 1000, -5, 5, seed=2, flags=ev.evox.FLAG_NO_SMALL | ev.evox.FLAG_NO_MID)
pso.step("ackley", 3)                    # multi-CTA generation kernel + grid argmin
pso.best()
for p, N, D in (("griewank", 340_000, 100), ("rosenbrock", 140_000, 250), ("ackley", 34_000, 1000)):
    pso = ev.PSO(N, D, -5, 5, seed=2)    # > 2^25 elements: flat tiles (short rows) / wave grid + prefetch
    pso.step(p, 2)
    pso.best()
    pso.close()
for p in ("sphere", "ackley", "rosenbrock"):
    pso = ev.PSO(3001, 1000, -5, 5, seed=2)  # cooperative kernel with the flat tail tiles
    pso.step(p, 3)
    pso.best()
    pso.close()
pso = ev.PSO(8200, 4100, -5, 5, seed=2)  # > 2^25 elements, CTA-per-row: wave grid + k_pso_fin
pso.step("rosenbrock", 2)
pso.best()
pso.close()
for D in (100, 20000):                   # peer exchange: key-first k_pso_fin (5 CTAs at 20000)
    hs = [ev.PSO(64, D, -5, 5, seed=3, rank=r, world=2, stream=torch.cuda.Stream())
          for r in range(2)]
    boxes = [h.mailbox()[0] for h in hs]
    for h in hs:
        h.connect_local(boxes)
    for h in hs:
        h.step("sphere", 3)
    for h in hs:
        h.sync()
    for h in hs:
        h.best()
des = [ev.DE(40, 33, -5, 5, seed=3, rank=r, world=2, stream=torch.cuda.Stream()) for r in range(2)]
bases = [h.state_base() for h in des]
for h in des:
    h.connect_local(bases)
for h in des:
    h.step("ackley", 2)
for h in des:
    h.sync()
for h in des:
    h.view("X")                          # gathered without touching the peer-read state
print("sanitize run ok")
