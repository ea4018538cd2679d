for rep in 1 2 3; do
  for K in 512 100; do
    echo "== K $K" >> gpurun_out/c1_check.log
    python bench.py --config C1 --steps $K --warmup 10 --reps 5 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*\|"sm_mhz": [0-9]*' | tr '\n' ' ' >> gpurun_out/c1_check.log
    echo >> gpurun_out/c1_check.log
  done
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,pci.bus_id --format=csv >> gpurun_out/c1_check.log
