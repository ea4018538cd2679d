for rep in 1 2; do
for f in 0 1 2; do
  echo "== flags $f" >> gpurun_out/c1_flags.log
  VTI_SMALL_FLAGS=$f python bench.py --config C1 --steps 320 --warmup 10 --reps 5 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/c1_flags.log
done
done
VTI_SMALL_FLAGS=1 timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_n4_gpu.py -q -x > gpurun_out/c1_flags_tests.log 2>&1; echo rc=$? >> gpurun_out/c1_flags_tests.log
