#!/bin/bash
# ncu --set full of the default adjoint kernels (each command exits 0 without ncu first); raw + details CSV kept
mkdir -p gpurun_out
for spec in "C2 32 ^k_adj_tma$" "N1 32 ^k_adj_tma2$" "C2 64 ^k_adj_tma2$" "N1 64 ^k_adj_tma2$"; do
  set -- $spec
  B="python tools/adjoint_rate.py --config $1 --precision $2 --steps 4 --warmup 3"
  rep=gpurun_out/prof_adj_$1_f$2
  $B > gpurun_out/adj_plain_$1_$2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"$3" -s 4 -c 1 -o $rep $B > gpurun_out/adj_ncu_$1_$2.log 2>&1; echo "ncu $1 f$2 rc=$?"
  ncu -i $rep.ncu-rep --page raw --csv > ${rep}_raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page details --csv > ${rep}_details.csv 2>/dev/null
  rm -f $rep.ncu-rep
done


