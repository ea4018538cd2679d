# C1 small-grid A/B: tile height of the small-grid kernel x one-step (graphs + PDL) vs multi-step
for rep in 1 2; do
for v in "" "VTI_SMALL_TY=32" "VTI_MULTI=1" "VTI_MULTI=1 VTI_SMALL_TY=32"; do
  echo "== [$v]" >> gpurun_out/c1_ab.log
  env $v python bench.py --config C1 --steps 200 --warmup 10 --reps 3 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*\|"tile_y": [0-9]*\|"steps_per_launch": [0-9]*\|"grid": [0-9]*' | tr '\n' ' ' >> gpurun_out/c1_ab.log
  echo >> gpurun_out/c1_ab.log
done
done
