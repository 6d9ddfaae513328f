# round-2 GPU check: the whole -m gpu suite, bench lines, and the 2-rank same-GPU flow
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu.log
for c in H C5 C4g; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 20 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err; done
for c in H C5; do EVOX_BENCH_SAME_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/b2_$c.json 2>gpurun_out/b2_$c.err; done
python - <<'P'
import json
for f in ["b_H", "b_C5", "b_C4g", "b2_H", "b2_C5"]:
    try:
        d = json.loads([l for l in open(f"gpurun_out/{f}.json") if l.startswith("{")][-1])
        print(f, round(d["value"], 2), round(d["roofline"]["frac"], 4), d["roofline"]["kernel"], d.get("exchange"), d["e2e"].get("breakdown_ms"))
    except Exception as e:
        print(f, "ERR", e)
P
