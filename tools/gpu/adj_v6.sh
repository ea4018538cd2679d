#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/adj_v6.log
: > $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
for c in C2 C3 C5; do ARGS="--config $c --precision 64"; r X=$c VTI_ADJ_TMA_TY=16; r X=$c; done
echo done >> $O
