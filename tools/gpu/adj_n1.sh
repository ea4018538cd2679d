#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/adj_n1.log
: > $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
ARGS="--config N1"
for st in 2 3 4; do r VTI_ADJ_TMA_ST=$st; r VTI_ADJ_TMA_ST=$st VTI_ADJ_CHAIN=0; done
ARGS="--config C2 --precision 64"; r VTI_ADJ_CHAIN=0; r X=1
ARGS="--config C3 --precision 64"; r VTI_ADJ_CHAIN=0
ncu --set full --clock-control none -k regex:k_adj_tma2 -s 4 -c 1 -o gpurun_out/ncu_adj_n1 python tools/adjoint_rate.py --config N1 --steps 3 --warmup 3 > gpurun_out/ncu_adj_n1.txt 2>&1
echo done >> $O
