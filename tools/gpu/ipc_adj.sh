#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/ipc_adj.log
timeout 900 python -m pytest tests/test_ipc_gpu.py tests/test_adjoint_gpu.py tests/test_peer_gpu.py tests/test_multigpu_gpu.py -q -x > $O 2>&1; echo "pytest rc=$?" >> $O
