#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/adj_graph2.log
: > $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
for p in 32 64; do ARGS="--config C1 --steps 200 --warmup 40 --precision $p"; r X=C1-$p; r X=C1-$p VTI_GRAPH=0; r X=C1-$p VTI_GRAPH=0 VTI_PDL=0; done
echo done >> $O
