"""Per-kernel SASS instruction counts of libevox.so (static, from cuobjdump -sass): the memory
instructions that prove the access path (LDG/STG .128 with evict-first hints, UBLKPF = the
cp.async.bulk.prefetch.L2 bulk prefetch, UBLKCP = cp.async.bulk copies into shared memory,
SYNCS = mbarrier ops), warp shuffles, global atomics and totals.

    python scripts/sass_summary.py [libevox.so] > profiles/sass_summary.txt
"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2301_12457_b200/libevox.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m and cur:
        funcs[cur].append(m.group(1))


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return out.stdout.splitlines()


# the kernels the bench configs run (first matching instantiation of each family)
want = [("k_pso_gen_wave<1, evox::(anonymous namespace)::Geom<32, 1, 2, false>, true, true>", "H: k_pso_gen_wave<ackley>, warp per row, tile prefetch"),
        ("k_pso_gen_flat<4, evox::(anonymous namespace)::Geom<4, 1, 4, false>, true>", "C4r: k_pso_gen_flat<rosenbrock>, flat tiles of 64 rows"),
        ("k_pso_gen_flat<3, evox::(anonymous namespace)::Geom<4, 1, 4, false>, true>", "C4g: k_pso_gen_flat<griewank>, flat tiles of 64 rows"),
        ("k_pso_gen_wave<1, evox::(anonymous namespace)::Geom<32, 8, 3, true>, true, false>", "C5: k_pso_gen_wave<ackley>, CTA per row"),
        ("k_pso_run_mid<1, evox::(anonymous namespace)::Geom<32, 1, 4, true>, true>", "C2: k_pso_run_mid<ackley> (+ tail tiles)"),
        ("k_pso_gen<3, evox::(anonymous namespace)::Geom<32, 1, 4, true>, true>", "persistent row walk: k_pso_gen<griewank>, warp per row"),
        ("k_pso_gen_tma<1, true>", "opt-in: k_pso_gen_tma<ackley> (EVOX_FLAG_TMA)"),
        ("k_pso_fin(", "k_pso_fin (gbest publication / key-first exchange)"),
        ("k_cso_gen<2, evox::(anonymous namespace)::Geom<8, 1, 4, true>, true>", "C3: k_cso_gen<rastrigin>"),
        ("k_de_gen_flat<0, evox::(anonymous namespace)::Geom<4, 1, 4, false>, true>", "D1: k_de_gen_flat<sphere>"),
        ("k_de_gen<1, evox::(anonymous namespace)::Geom<32, 1, 4, true>, true>", "D2: k_de_gen<ackley>"),
        ("k_eval<1, evox::(anonymous namespace)::Geom<32, 1, 4, true> >", "EH: k_eval<ackley>")]
dem = dict(zip(funcs, demangle(list(funcs))))
classes = [("LDG.128", r"^LDG\.E(\.\w+)*\.128"), ("LDG.128 evict-first", r"^LDG\.E\.EF(\.\w+)*\.128"),
           ("STG.128", r"^STG\.E(\.\w+)*\.128"), ("STG.128 evict-first", r"^STG\.E\.EF(\.\w+)*\.128"),
           ("LDG other", r"^LDG(?!.*\.128)"), ("STG other", r"^STG(?!.*\.128)"),
           ("LDS", r"^LDS"), ("STS", r"^STS"), ("UBLKPF", r"^UBLKPF"), ("UBLKCP", r"^UBLKCP"),
           ("SYNCS", r"^SYNCS"), ("SHFL", r"^SHFL"), ("ATOMG/REDG", r"^(ATOMG|RED)"),
           ("IMAD.WIDE.U32 / IMAD.HI", r"^IMAD\.(WIDE|HI)"), ("MUFU", r"^MUFU"),
           ("total", r".")]
print("# Static SASS of paper_2301_12457_b200/libevox.so (cuobjdump -sass), per kernel:")
print("# instruction counts by class (mnemonic regex on the opcode).  Dynamic per-element cost at H")
print("# (ncu smsp__inst_executed.sum, profiles/r02_ncu_full_H.txt): 2.168e9 warp instructions per")
print("# launch x 32 lanes / 1e9 elements = 69.4 lane-instructions per element-generation.")
for key, label in want:
    hits = [f for f in funcs if key in dem[f]]
    if not hits:
        print(f"\n## {label}: not found ({key})")
        continue
    ops = funcs[hits[0]]
    print(f"\n## {label}\n#  {dem[hits[0]][:150]}")
    for name, rx in classes:
        n = sum(1 for o in ops if re.search(rx, o))
        print(f"   {name:26s} {n}")
