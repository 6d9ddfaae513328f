# Round-end evidence on one GPU: the -m gpu suite, smoke(), every generation kernel under ncu --set full
# (raw CSV exported on the box), the H launch list, and every bench line (with cool-downs).
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
bash scripts/gpu_ncu_all.sh ${NCU_TAG:-r02c} > gpurun_out/ncu_all.log 2>&1; cat gpurun_out/ncu_all.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pso_run_mid -s 1 -c 1 -o /tmp/prof_c2c python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --sustained-s 0 > gpurun_out/ncu_c2c.log 2>&1; ncu -i /tmp/prof_c2c.ncu-rep --page raw --csv > gpurun_out/ncu_${NCU_TAG:-r02c}_C2_raw.csv
rm -f gpurun_out/bench_*; bash scripts/gpu_bench_all.sh
