#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/adj_v7.log
: > $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
ARGS="--config N1 --precision 64"; r X=N1 VTI_ADJ_TMA_TY=4 VTI_ADJ_TMA_ST=2; r X=N1 VTI_ADJ_TMA_TY=4 VTI_ADJ_TMA_ST=3; r X=N1
echo done >> $O
