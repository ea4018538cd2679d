for rep in 1 2; do
for v in "" "VTI_SMALL_PX=4"; do
  for K in 512 100; do
  echo "== [$v] K $K" >> gpurun_out/c1_px2.log
  env $v python bench.py --config C1 --steps $K --warmup 10 --reps 5 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/c1_px2.log
  done
done
done
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_n4_gpu.py tests/test_multistep_gpu.py -q -x > gpurun_out/c1_px2_tests.log 2>&1; echo rc=$? >> gpurun_out/c1_px2_tests.log
for cfg in "C5" "C3"; do echo "== small ragged via tests ok" > /dev/null; done
