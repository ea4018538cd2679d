for rep in 1 2; do
for v in "" "VTI_TY=8 VTI_STAGES=2" "VTI_TY=6"; do
  echo "== [$v]" >> gpurun_out/n1f64_minb2.log
  env $v python bench.py --config N1 --precision 64 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*\|"tile_y": [0-9]*' | tr '\n' ' ' >> gpurun_out/n1f64_minb2.log
  echo >> gpurun_out/n1f64_minb2.log
done
done
