#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/adj_zc.log
: > $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
for p in 32 64; do ARGS="--config C1 --steps 200 --warmup 10 --precision $p"; for z in 1 2 4 8; do r X=C1-$p VTI_ADJ_ZCHUNK=$z; done; r X=C1-$p VTI_ADJ_ZCHUNK=2 VTI_ADJ_TMA_TY=16; done
echo done >> $O
