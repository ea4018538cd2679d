for K in 100 320 512; do
  echo "== K $K" >> gpurun_out/c1_g2.log
  python bench.py --config C1 --steps $K --warmup 10 --reps 5 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/c1_g2.log
done
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_n4_gpu.py tests/test_multistep_gpu.py tests/test_bench_contract.py -q -x > gpurun_out/c1_g2_tests.log 2>&1; echo rc=$? >> gpurun_out/c1_g2_tests.log
