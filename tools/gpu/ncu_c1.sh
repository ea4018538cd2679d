# ncu --set full of the multi-step C1 kernel (one launch = one timed region of K steps)
ncu --set full --import-source on --clock-control none -k regex:vti_small_multi -c 1 -o gpurun_out/ncu_c1_multi \
  python bench.py --config C1 --steps 200 --warmup 10 --reps 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c1_multi.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:vti_small_kernel -s 20 -c 1 -o gpurun_out/ncu_c1_small \
  env VTI_MULTI=0 python bench.py --config C1 --steps 200 --warmup 10 --reps 1 --no-e2e --no-cpu-baseline >> gpurun_out/ncu_c1_multi.log 2>&1
