for rep in 1 2; do
for v in "" "VTI_PTILE_LDG=1"; do
  echo "== [$v]" >> gpurun_out/c1_ptile.log
  env $v python bench.py --config C1 --steps 512 --warmup 10 --reps 5 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/c1_ptile.log
done
done
VTI_PTILE_LDG=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_n4_gpu.py -q -x > gpurun_out/c1_ptile_tests.log 2>&1; echo rc=$? >> gpurun_out/c1_ptile_tests.log
