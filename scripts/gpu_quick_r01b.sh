mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "griewank_table or fused_fitness or eval_parity" -p no:cacheprovider > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for c in E5-griewank EH-griewank; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; done
EVOX_NO_HTAB=1 timeout 300 python bench.py --config E5-griewank --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b_E5-griewank_notab.json 2>&1
for c in C4g C5 H; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; done
