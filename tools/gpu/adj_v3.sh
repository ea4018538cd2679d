#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/adj_v3.log
: > $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
ARGS="--config C3"; r X=C3 VTI_ADJ_TMA_TY=8 VTI_ADJ_FORM=1; r X=C3
ARGS="--config C5"; r X=C5 VTI_ADJ_TMA_TY=8 VTI_ADJ_FORM=1; r X=C5
ARGS="--config C2 --precision 64"; r X=C2-f64
ARGS="--config C3 --precision 64"; r X=C3-f64 VTI_ADJ_TMA_PX=4 VTI_ADJ_TMA_ST=3; r X=C3-f64 VTI_ADJ_TMA_MINB=2
ARGS="--config C5 --precision 64"; r X=C5-f64 VTI_ADJ_TMA_PX=4
timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x >> $O 2>&1; echo "pytest rc=$?" >> $O
echo done >> $O
