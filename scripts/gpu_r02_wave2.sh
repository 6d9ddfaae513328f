timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "wave or full_size or mid_kernel or graphed" > gpurun_out/r02_wave_pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/r02_wave_pytest.log
bash scripts/gpu_r02_ab.sh "H C4g C4r C5" "base w0 wu4 wu2 w2" 1
