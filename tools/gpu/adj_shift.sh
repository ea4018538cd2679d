#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/adj_shift.log
: > $O
timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x >> $O 2>&1; echo "pytest rc=$?" >> $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
ARGS="--config N1"; r X=N1; r X=N1 VTI_ADJ_CHAIN=0; r X=N1 VTI_ADJ_TMA_ST=4; r X=N1 VTI_ADJ_FORM=1
ARGS="--config C5"; r X=C5; r X=C5 VTI_ADJ_FORM=2
ARGS="--config C2"; r X=C2
ARGS="--config C3"; r X=C3
for c in C2 C3 C5 N1; do ARGS="--config $c --precision 64"; r X=$c-f64; done
echo done >> $O
