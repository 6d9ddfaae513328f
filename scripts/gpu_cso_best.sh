#!/bin/bash
# CSO best() single-rank shortcut: full GPU suite + C3 line (e2e).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/csob_tests.log 2>&1; echo rc=$? >> gpurun_out/csob_tests.log
timeout 600 python bench.py --config C3 > gpurun_out/csob_C3.json 2> gpurun_out/csob_C3.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/csob_smoke.log 2>&1; echo smoke=$? >> gpurun_out/csob_smoke.log
