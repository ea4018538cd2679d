for rep in 1 2; do
for g in 32 64 128 256; do
  echo "== graph steps $g" >> gpurun_out/c1_gs.log
  VTI_GRAPH_STEPS=$g python bench.py --config C1 --steps 512 --warmup 10 --reps 5 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/c1_gs.log
done
done
