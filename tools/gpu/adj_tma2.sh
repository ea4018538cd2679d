#!/bin/bash
# TMA adjoint forms: parity, then rates per config and form (VTI_ADJ_FORM, VTI_ADJ_TMA_TY).
mkdir -p gpurun_out
O=gpurun_out/adj_tma2.log
: > $O
timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x >> $O 2>&1; echo "pytest rc=$?" >> $O
r() { echo "[$*]" >> $O; env "$@" timeout 300 python tools/adjoint_rate.py $ARGS 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; }
for c in C2 C5; do
  ARGS="--config $c"
  r X=$c VTI_ADJ_FORM=1 VTI_ADJ_TMA_TY=8; r X=$c VTI_ADJ_FORM=1 VTI_ADJ_TMA_TY=16; r X=$c VTI_ADJ_FORM=2
done
ARGS="--config C3"; r X=C3 VTI_ADJ_FORM=1 VTI_ADJ_TMA_TY=8; r X=C3 VTI_ADJ_FORM=1 VTI_ADJ_TMA_TY=16; r X=C3 VTI_ADJ_FORM=2
ARGS="--config N1"; r X=N1 VTI_ADJ_FORM=2; r X=N1 VTI_ADJ_FORM=1
for c in C2 C3 C5 N1; do
  ARGS="--config $c --precision 64"
  r X=$c-f64 VTI_ADJ_FORM=2 VTI_ADJ_TMA_PX=2; r X=$c-f64 VTI_ADJ_FORM=2 VTI_ADJ_TMA_PX=4; r X=$c-f64 VTI_ADJ_FORM=1
done
echo done >> $O
