#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/adj_more.log
timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x > $O 2>&1; echo "pytest rc=$?" >> $O
VTI_LAYOUT=yzx timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x >> $O 2>&1; echo "pytest yzx rc=$?" >> $O
VTI_ADJ_TMA=0 timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x >> $O 2>&1; echo "pytest cp.async forms rc=$?" >> $O
VTI_ADJ_CHAIN=0 timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x >> $O 2>&1; echo "pytest unchained rc=$?" >> $O
