# N1 fp64: two rows per thread (RPT = 2) against the default, twice
for rep in 1 2; do
for v in "" "VTI_TY=8 VTI_RPT=2" "VTI_TY=12 VTI_RPT=2" "VTI_TY=16 VTI_RPT=2"; do
  echo "== [$v]" >> gpurun_out/n1f64_rpt2.log
  env $v python bench.py --config N1 --precision 64 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | grep -o '"value": [0-9.]*\|"tile_y": [0-9]*\|"rows_per_thread": [0-9]*' | tr '\n' ' ' >> gpurun_out/n1f64_rpt2.log
  echo >> gpurun_out/n1f64_rpt2.log
done
done
