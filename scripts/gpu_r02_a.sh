set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./scripts/micro/ring > gpurun_out/r02_micro_ring.txt 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_H.json 2>gpurun_out/b_H.err
EVOX_NP=4 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_H_np4.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/r02_micro_ring.txt
