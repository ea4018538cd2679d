#!/bin/bash
# programmatic dependent launch for the TMA adjoint kernels: parity, then rates with / without
mkdir -p gpurun_out
O=gpurun_out/adj_pdl.log
: > $O
timeout 900 python -m pytest tests/test_adjoint_gpu.py tests/test_ipc_gpu.py -q -x >> $O 2>&1; echo "pytest rc=$?" >> $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
for c in C1 C2 N1; do ARGS="--config $c --steps 100"; r X=$c; r X=$c VTI_PDL=0; done
ARGS="--config C1 --steps 100 --precision 64"; r X=C1-f64; r X=C1-f64 VTI_PDL=0
echo done >> $O
