# usage: bash tools/profile_some.sh "C5 32" "N1 32" ...  (ncu --set full of the step kernel, CSV exports)
set -u
out=gpurun_out
for spec in "$@"; do
  set -- $spec
  B="python bench.py --config $1 --precision $2 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline"
  rep=$out/prof_$1_f$2
  $B > $out/plain_$1_$2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:vti_step_kernel -s 3 -c 1 -o $rep $B > $out/ncu_$1_$2.log 2>&1; echo "ncu $1 f$2 rc=$?"
  ncu -i $rep.ncu-rep --page raw --csv > ${rep}_raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page details --csv > ${rep}_details.csv 2>/dev/null
  rm -f $rep.ncu-rep
done
