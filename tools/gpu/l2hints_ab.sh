# L2 cache-policy A/B: evict_first on the read-once TMA streams (bit 0), streaming stores (bit 1)
for rep in 1 2; do
for cfg in C4 C5 C3 C2; do
for hint in 0 1 2 3; do
  echo "== $cfg hints $hint" >> gpurun_out/l2hints.log
  VTI_L2_HINTS=$hint python bench.py --config $cfg --steps 10 --warmup 3 --reps 5 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*\|"sm_mhz": [0-9]*' | tr '\n' ' ' >> gpurun_out/l2hints.log
  echo >> gpurun_out/l2hints.log
done
done
done
