for rep in 1 2; do
for v in "" "VTI_MULTI=1 VTI_MULTI_MODE=32" "VTI_MULTI=1 VTI_MULTI_MODE=48"; do
  echo "== [$v]" >> gpurun_out/multi_barrier.log
  env $v timeout 120 python bench.py --config C1 --steps 512 --warmup 10 --reps 5 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/multi_barrier.log
done
done
VTI_MULTI_MODE=48 timeout 600 python -m pytest tests/test_multistep_gpu.py -q > gpurun_out/multi_barrier_tests.log 2>&1; echo rc=$? >> gpurun_out/multi_barrier_tests.log
