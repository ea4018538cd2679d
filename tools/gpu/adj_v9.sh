#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/adj_v9.log
: > $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
ARGS="--config N1"; r X=N1; r X=N1 VTI_ADJ_TMA_TY=4; r X=N1 VTI_ADJ_TMA_PX=2 VTI_ADJ_TMA_TY=8
VTI_ADJ_TMA_TY=4 timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x -k "12-8-32 or 12, 8, 32" >> $O 2>&1; echo "pytest ty4 rc=$?" >> $O
echo done >> $O
