# one ncu --set full capture of a generation kernel, exported to text on the box (the
# .ncu-rep stays behind): bash scripts/gpu_r02_ncu.sh <tag> <config> <kernel regex>
tag=$1; cfg=$2; k=$3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o /tmp/prof_$tag python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_$tag.log 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_${tag}_raw.csv 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page source --csv > gpurun_out/ncu_${tag}_source.csv 2>&1
ncu -i /tmp/prof_$tag.ncu-rep --page details --csv > gpurun_out/ncu_${tag}_details.csv 2>&1
ls -la gpurun_out/ncu_${tag}*
