# N1 fp64 variant A/B (1000-step config timed 20 steps x 5 regions each), twice
for rep in 1 2; do
for v in "default" "1 8 4" "1 8 3" "1 6 5" "1 4 4"; do
  set -- $v
  if [ "$1" = default ]; then env=""; else env="VTI_PX=$1 VTI_TY=$2 VTI_STAGES=$3"; fi
  echo "== $v" >> gpurun_out/n1f64_ab.log
  env $env python bench.py --config N1 --precision 64 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*\|"tile_y": [0-9]*\|"points_per_thread": [0-9]*' | tr '\n' ' ' >> gpurun_out/n1f64_ab.log
  echo >> gpurun_out/n1f64_ab.log
done
done
