#!/bin/bash
# Every bench line on 1 GPU (default steps/warm-up, CPU oracle baseline included) -> gpurun_out/bench_<cfg>.json.
# Each line ends with its own ~1.5 s sustained (power-capped) window, so the next config starts only after a
# cool-down: the board's power limit averages over a window and would otherwise cap the next burst measurement.
mkdir -p gpurun_out
for c in ${@:-H C1 C2 C3 C4g C4r C5 D1 D2}; do
  sleep ${COOLDOWN_S:-20}
  timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
for c in EH-sphere EH-ackley EH-rastrigin EH-griewank EH-rosenbrock E5-sphere E5-ackley E5-rastrigin E5-griewank E5-rosenbrock; do
  [ -n "$1" ] && break
  timeout 600 python bench.py --config $c --e2e-steps 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
ls gpurun_out/bench_*.json | wc -l
