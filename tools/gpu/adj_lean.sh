#!/bin/bash
# LEAN one-pass adjoint (s1 in place, psi^{m+1} from HBM): parity, then rates
mkdir -p gpurun_out
O=gpurun_out/adj_lean.log
: > $O
VTI_ADJ_LEAN=1 timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x -k "32" >> $O 2>&1; echo "pytest lean px2 rc=$?" >> $O
VTI_ADJ_LEAN=1 VTI_ADJ_TMA_PX=4 timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x -k "32" >> $O 2>&1; echo "pytest lean px4 rc=$?" >> $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
for c in C2 C3 C5; do ARGS="--config $c"; r X=$c VTI_ADJ_LEAN=1; r X=$c VTI_ADJ_LEAN=1 VTI_ADJ_TMA_PX=4; r X=$c; done
echo done >> $O
