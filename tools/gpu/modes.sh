# the parity / peer / N4 / fp64 / adjoint suites under the non-default modes
for v in "VTI_LAYOUT=yzx" "VTI_GRAPH=0" "VTI_SMALL_DIRECT=0" "VTI_ALIGN=0" "VTI_FUSED_STEP=1"; do
  env $v timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_peer_gpu.py tests/test_n4_gpu.py tests/test_fp64_gpu.py tests/test_adjoint_gpu.py -q -p no:cacheprovider > gpurun_out/modes_tmp.log 2>&1
  echo "[$v] rc=$? $(tail -n 1 gpurun_out/modes_tmp.log)" >> gpurun_out/modes.log
  grep -E "^FAILED" gpurun_out/modes_tmp.log | head -5 >> gpurun_out/modes.log
done
