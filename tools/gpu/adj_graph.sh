#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/adj_graph.log
: > $O
timeout 900 python -m pytest tests/test_adjoint_gpu.py tests/test_ipc_gpu.py -q -x >> $O 2>&1; echo "pytest rc=$?" >> $O
VTI_GRAPH=0 timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x -k graph >> $O 2>&1; echo "pytest nograph rc=$?" >> $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
for p in 32 64; do ARGS="--config C1 --steps 100 --precision $p"; r X=C1-$p; r X=C1-$p VTI_GRAPH=0; done
ARGS="--config C2 --steps 20"; r X=C2
echo done >> $O
