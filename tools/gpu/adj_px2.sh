#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/adj_px2.log
: > $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
for c in C2 C3 C5; do ARGS="--config $c"; r X=$c VTI_ADJ_FORM=1 VTI_ADJ_TMA_PX=2; r X=$c; done
VTI_ADJ_TMA_PX=2 timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x >> $O 2>&1; echo "pytest px2 rc=$?" >> $O
echo done >> $O
