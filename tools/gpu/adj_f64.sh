for c in C2 C3 C5 N1; do
  for v in "VTI_ADJ_TWO_PASS=1" "VTI_ADJ_TWO_PASS=0"; do
    echo "[$v]" >> gpurun_out/adj_f64.log; env $v python tools/adjoint_rate.py --config $c --precision 64 2>&1 | cut -c1-140 >> gpurun_out/adj_f64.log
  done
done
