for rep in 1 2; do
for v in "VTI_SMALL=0" "" "VTI_SMALL_DIRECT=0"; do
  echo "== [$v]" >> gpurun_out/c1_f64.log
  env $v python bench.py --config C1 --precision 64 --steps 512 --warmup 10 --reps 5 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*\|"small_kernel": [0-9]' | tr '\n' ' ' >> gpurun_out/c1_f64.log
  echo >> gpurun_out/c1_f64.log
done
done
timeout 900 python -m pytest tests/test_fp64_gpu.py tests/test_parity_gpu.py tests/test_n4_gpu.py -q -x > gpurun_out/c1_f64_tests.log 2>&1; echo rc=$? >> gpurun_out/c1_f64_tests.log
