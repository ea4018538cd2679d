#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --config N1 --precision 64 --steps 4 --warmup 3 --reps 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/n1f64_plain.log 2>&1 && ncu --set full --clock-control none -k regex:"^vti_step_kernel$" -s 3 -c 1 -o gpurun_out/prof_n1f64 $B > gpurun_out/n1f64_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_n1f64.ncu-rep --page raw --csv > gpurun_out/prof_n1f64_raw.csv 2>/dev/null
rm -f gpurun_out/prof_n1f64.ncu-rep
