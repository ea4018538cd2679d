# C1: TMA-staged small-grid kernel vs the direct-load form, twice; then parity with the direct form
for rep in 1 2; do
for v in "" "VTI_SMALL_DIRECT=1"; do
  echo "== [$v]" >> gpurun_out/c1_direct.log
  env $v python bench.py --config C1 --steps 320 --warmup 10 --reps 5 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/c1_direct.log
done
done
VTI_SMALL_DIRECT=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_n4_gpu.py tests/test_multistep_gpu.py -q -x > gpurun_out/c1_direct_tests.log 2>&1; echo rc=$? >> gpurun_out/c1_direct_tests.log
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_n4_gpu.py -q -x >> gpurun_out/c1_direct_tests.log 2>&1; echo rc=$? >> gpurun_out/c1_direct_tests.log
