#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/adj_f64b.log
: > $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
for c in C2 C3 C5; do ARGS="--config $c --precision 64"; r X=$c VTI_ADJ_TMA_MINB=2; r X=$c; done
ARGS="--config C2 --precision 64"; r X=C2 VTI_ADJ_TMA_ST=3
timeout 600 python -m pytest tests/test_multigpu_gpu.py tests/test_ipc_gpu.py -q >> $O 2>&1; echo "pytest rc=$?" >> $O
VTI_ADJ_TMA_MINB=2 timeout 600 python -m pytest tests/test_adjoint_gpu.py -q -x -k "64" >> $O 2>&1; echo "pytest minb2 rc=$?" >> $O
echo done >> $O
