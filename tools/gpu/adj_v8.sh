#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/adj_v8.log
: > $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
ARGS="--config N1 --precision 64"; r X=N1; r X=N1 VTI_ADJ_TMA_TY=4 VTI_ADJ_TMA_ST=4
for c in C2 C3 C5; do ARGS="--config $c --precision 64"; r X=$c VTI_ADJ_TMA_TY=4; r X=$c; done
timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x -k "64" >> $O 2>&1; echo "pytest f64 rc=$?" >> $O
VTI_ADJ_TMA_TY=4 timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x -k "64" >> $O 2>&1; echo "pytest f64 ty4 rc=$?" >> $O
echo done >> $O
