# GPU check: the whole -m gpu suite, the sanitizers on every kernel family, bench lines
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_run.py > gpurun_out/sanitizer_$tool.log 2>&1; echo "$tool rc=$?"; tail -2 gpurun_out/sanitizer_$tool.log
done
for c in ${BENCH_CONFIGS:-H}; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err; done
python - <<'P'
import json, glob
for f in sorted(glob.glob("gpurun_out/b_*.json")):
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
        print(f, round(d["value"], 2), round(d["roofline"]["frac"], 4), d["roofline"]["kernel"], round(d["e2e"]["value"], 2), d["e2e"].get("breakdown_ms"))
    except Exception as e:
        print(f, "ERR", e)
P
python scripts/setup_probe.py 2>&1 | tail -8
