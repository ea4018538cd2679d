for v in "" "VTI_ADJ_TWO_PASS=1" "VTI_ADJ_TWO_PASS=0"; do env $v timeout 600 python -m pytest tests/test_adjoint_gpu.py -q > /dev/null 2>&1; echo "[$v] tests rc=$?" >> gpurun_out/adj_v2.log; done
for c in N1 C2 C3; do
  for v in "VTI_ADJ_TWO_PASS=1" "VTI_ADJ_TWO_PASS=0"; do
    echo "[$v]" >> gpurun_out/adj_v2.log; env $v python tools/adjoint_rate.py --config $c 2>&1 | cut -c1-120 >> gpurun_out/adj_v2.log
  done
done
