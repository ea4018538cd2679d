#!/bin/bash
mkdir -p gpurun_out
B="python tools/adjoint_rate.py --config C3 --steps 4 --warmup 3"
rep=gpurun_out/prof_adj_C3_f32
$B > gpurun_out/adj_plain_C3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"^k_adj_tma$" -s 4 -c 1 -o $rep $B > gpurun_out/adj_ncu_C3.log 2>&1; echo "ncu rc=$?"
ncu -i $rep.ncu-rep --page raw --csv > ${rep}_raw.csv 2>/dev/null
ncu -i $rep.ncu-rep --page source --csv > ${rep}_source.csv 2>/dev/null
rm -f $rep.ncu-rep
