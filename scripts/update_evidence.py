"""Copy a round-end evidence run (scripts/gpu_final.sh) from gpurun_out/ into profiles/: bench lines,
ncu --set full summaries + profiles/ncu_summary.json, the H launch list, and the DESIGN.md results
tables.     python scripts/update_evidence.py <ncu tag, e.g. r02d>"""
import glob
import json
import os
import subprocess
import sys

tag = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.chdir(ROOT)
for f in glob.glob("gpurun_out/bench_*.json"):
    c = os.path.basename(f)[len("bench_"):-len(".json")]
    lines = [l for l in open(f) if l.startswith("{")]
    if lines:
        open(f"profiles/r02_bench_{c}.json", "w").write(lines[-1])
algo = {"H": 20 * 1e6 * 1000 + 10 * 1e6, "C3": 10 * 1e5 * 1000 + 6 * 1e5, "C4g": 20 * 1e8 + 10 * 1e6,
        "C4r": 20 * 1e8 + 10 * 1e6, "C5": 20 * 1e4 * 1e5 + 10 * 1e4, "D1": 20 * 1e8 + 13 * 1e6,
        "D2": 20 * 1e9 + 13 * 1e6, "EH-ackley": 4 * 1e9 + 4 * 1e6, "E5-griewank": 4 * 1e9 + 4 * 1e4,
        "C2": 200100000}
summ = json.load(open("profiles/ncu_summary.json"))
for c, a in algo.items():
    txt = subprocess.run(["python", "scripts/ncu_summary.py", f"gpurun_out/ncu_{tag}_{c}_raw.csv"],
                         capture_output=True, text=True).stdout
    kn = rd = wr = None
    for line in txt.splitlines():
        if line.startswith("Kernel Name"):
            kn = line[60:].strip()
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if line.startswith(key):
                v, u = line.split()[1:3]
                val = float(v) * (1e9 if u == "Gbyte" else 1e6)
                rd, wr = (val, wr) if key.endswith("read.sum") else (rd, val)
    per = 2 if c == "C2" else 1
    name = "C2-mid" if c == "C2" else c
    if c == "C2":
        txt += ("# 1 launch of k_pso_run_mid = 2 generations (bench --steps 2); per generation: DRAM %.1f MB "
                "(%.3f of the 200.1 MB algorithmic: the 120 MB state is L2-sized)\n" % ((rd + wr) / 2 / 1e6, (rd + wr) / 2 / a))
    open(f"profiles/r02_ncu_full_{name}.txt", "w").write(txt)
    summ[c] = {"kernel": kn, "dram_bytes_per_launch": (rd + wr) / per, "algorithmic_bytes_per_launch": int(a),
               "source": f"profiles/r02_ncu_full_{name}.txt (ncu --set full --clock-control none, 1 launch at the "
                         f"bench config, round 2 closing kernels{'; per generation of a 2-generation launch' if c == 'C2' else ''}; "
                         "default --cache-control all flushes caches before the launch)"}
json.dump(summ, open("profiles/ncu_summary.json", "w"), indent=1)
lc = f"gpurun_out/launches_{tag}_H.csv"
if os.path.exists(lc):
    subprocess.run(["cp", lc, "profiles/r02_launches_H.csv"])
    out = subprocess.run(["python", "scripts/summarize_launches.py", lc], capture_output=True, text=True).stdout
    open("profiles/r02_launches_H.txt", "w").write(
        "# H (PSO/Ackley 1e6 x 1000): ncu --metrics gpu__time_duration.sum --clock-control none launch list of "
        "bench.py --config H --steps 2 --warmup 1 (cold-cache, serialised; init/eval are one-off setup, the "
        "generation = k_pso_gen_wave + k_pso_fin)\n" + out)
names = {"H": "PSO/Ackley 1e6x1000 (headline)", "C1": "PSO/Sphere 100x10, 100 gens, seed 0",
         "C2": "PSO/Ackley 1e4x1000 (persistent cooperative kernel + tail tiles)", "C3": "CSO/Rastrigin 1e5x1000",
         "C4g": "PSO/Griewank 1e6x100 (flat tiles)", "C4r": "PSO/Rosenbrock 1e6x100 (flat tiles)",
         "C5": "PSO/Ackley 1e4x1e5", "D1": "DE/Sphere 1e6x100 (flat tiles)", "D2": "DE/Ackley 1e6x1000"}
rows = []
for c in ["H", "C1", "C2", "C3", "C4g", "C4r", "C5", "D1", "D2"]:
    d = json.loads(open(f"profiles/r02_bench_{c}.json").read())
    r, su = d["roofline"], d["sustained"]
    if c == "C1":
        frac, sf, ratio = "latency-bound (1 launch / n gens)", "–", "–"
    else:
        frac = f"{r['frac'] * 100:.1f}%"
        sf = f"{su['frac'] * 100:.1f}% @ {su['clocks']['sm_mhz']:.0f} MHz"
        ratio = f"{summ[c]['dram_bytes_per_launch'] / summ[c]['algorithmic_bytes_per_launch']:.3f}"
    rows.append(f"| {c} | {names[c]} | {d['value']:.4g} | {d['ms_per_step'] * 1e3:.1f} | {d['individual_dims_per_s']:.3g} | "
                f"{r['achieved']:.0f} | {frac} | {sf} | {ratio} | {d['e2e']['value']:.4g} | {d['cpu_baseline']['value']:.3g} |")
ev = []
for c in ["EH-sphere", "E5-sphere", "EH-ackley", "E5-ackley", "EH-rastrigin", "E5-rastrigin", "EH-griewank",
          "E5-griewank", "EH-rosenbrock", "E5-rosenbrock"]:
    d = json.loads(open(f"profiles/r02_bench_{c}.json").read())
    r = d["roofline"]
    fn, shape = c.split("-")[1], ("1e6x1000" if c.startswith("EH") else "1e4x1e5")
    ev.append(f"| {c} | {fn} {shape} | {d['value']:.4g} | {r['kernel_ms'] * 1e3:.0f} | {d['individual_dims_per_s']:.3g} | "
              f"{r['achieved']:.0f} | {r['frac'] * 100:.1f}% | {d['e2e']['value']:.3g} | {d['cpu_baseline']['value']:.3g} |")
s = open("DESIGN.md").read()
a = s.index("| id | workload | gen/s | µs/gen | individual-dims/s | achieved GB/s | of measured HBM peak (burst window) |")
a = s.index("\n", s.index("\n", a) + 1) + 1
b = s.index("\n\nRound 1 → round 2 (same metric", a)
s = s[:a] + "\n".join(rows) + s[b:]
a = s.index("| config | function, shape | populations/s | kernel µs |")
a = s.index("\n", s.index("\n", a) + 1) + 1
b = s.index("\n\n", a)
s = s[:a] + "\n".join(ev) + s[b:]
open("DESIGN.md", "w").write(s)
print("\n".join(rows))
