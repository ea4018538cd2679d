for m in 32 48; do
  VTI_MULTI_MODE=$m timeout 600 python -m pytest tests/test_multistep_gpu.py -q > gpurun_out/multi_barrier_tests_$m.log 2>&1; echo rc=$? >> gpurun_out/multi_barrier_tests_$m.log
done
for rep in 1 2; do
for v in "" "VTI_MULTI=1 VTI_MULTI_MODE=32" "VTI_MULTI=1 VTI_MULTI_MODE=48"; do
  for K in 512 100; do
  echo "== [$v] K $K" >> gpurun_out/multi_barrier2.log
  env $v timeout 120 python bench.py --config C1 --steps $K --warmup 10 --reps 5 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/multi_barrier2.log
  done
done
done
