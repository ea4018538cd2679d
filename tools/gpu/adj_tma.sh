#!/bin/bash
# The TMA adjoint kernel: parity (tests/test_adjoint_gpu.py) then rates vs the previous forms.
mkdir -p gpurun_out
O=gpurun_out/adj_tma.log
: > $O
timeout 600 python -m pytest tests/test_adjoint_gpu.py -q -x >> $O 2>&1; echo "pytest rc=$?" >> $O
for c in C2 C3 C5 N1; do
  echo "[tma $c]" >> $O; timeout 300 python tools/adjoint_rate.py --config $c >> $O 2>&1
done
echo "[tma C2 TY=8]" >> $O; VTI_ADJ_TMA_TY=8 timeout 300 python tools/adjoint_rate.py --config C2 >> $O 2>&1
echo "[old C2]" >> $O; VTI_ADJ_TMA=0 timeout 300 python tools/adjoint_rate.py --config C2 >> $O 2>&1
for c in C2 C3 C5 N1; do
  echo "[tma f64 $c]" >> $O; timeout 300 python tools/adjoint_rate.py --config $c --precision 64 >> $O 2>&1
done
echo done >> $O
