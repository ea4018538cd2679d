# C1 with the direct-load small-grid kernel: launch list and one --set full capture
B="python bench.py --config C1 --steps 64 --warmup 3 --reps 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/c1_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"vti" -c 200 --csv --log-file gpurun_out/launches_C1.csv $B > gpurun_out/ncu_c1_l.log 2>&1; echo "launches rc=$?"
$B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:vti_small -s 10 -c 1 -o gpurun_out/prof_C1_f32 $B > gpurun_out/ncu_c1_full.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_C1_f32.ncu-rep --page raw --csv > gpurun_out/prof_C1_f32_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_C1_f32.ncu-rep --page details --csv > gpurun_out/prof_C1_f32_details.csv 2>/dev/null
rm -f gpurun_out/prof_C1_f32.ncu-rep
