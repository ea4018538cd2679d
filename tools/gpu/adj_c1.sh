timeout 900 python -m pytest tests/test_adjoint_gpu.py tests/test_multistep_gpu.py -q -rA > gpurun_out/gputest_adj.log 2>&1; echo rc=$? >> gpurun_out/gputest_adj.log
VTI_SMALL_TY=32 timeout 600 python -m pytest tests/test_multistep_gpu.py tests/test_parity_gpu.py -q -k "small or c1 or ragged or chunked" > gpurun_out/gputest_ty32.log 2>&1; echo rc=$? >> gpurun_out/gputest_ty32.log
bash tools/gpu/c1_ab.sh
timeout 300 python -m pytest tests/test_n4_gpu.py -q -k snapshot >> gpurun_out/gputest_adj.log 2>&1
