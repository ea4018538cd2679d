for c in C2 C3 C5 N1; do
  for v in "VTI_ADJ_TWO_PASS=0 VTI_ADJ_TY=16" "VTI_ADJ_TWO_PASS=0 VTI_ADJ_TY=8" "VTI_ADJ_TWO_PASS=1"; do
    echo "[$v]" >> gpurun_out/adj_ty.log
    env $v python tools/adjoint_rate.py --config $c 2>&1 | cut -c1-120 >> gpurun_out/adj_ty.log
  done
done
VTI_ADJ_TWO_PASS=0 timeout 600 python -m pytest tests/test_adjoint_gpu.py -q > gpurun_out/adj_ty_tests.log 2>&1; echo rc=$? >> gpurun_out/adj_ty_tests.log
