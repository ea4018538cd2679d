# round-2 measurement pass: bench sweep (plain), launch list of the default (C4) line, and one
# ncu --set full capture of the step kernel per config (each command exits 0 without ncu first);
# reports exported to CSV on the box, .ncu-rep dropped (gpurun_out/ is capped at 64 MiB)
set -u
out=gpurun_out
for spec in "C4 32" "C2 32" "C3 32" "C5 32" "N1 32" "C1 32" "C2 64" "C3 64" "C5 64" "N1 64" "C1 64"; do
  set -- $spec
  python bench.py --config $1 --precision $2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $out/sweep_$1_f$2.json 2> $out/sweep_$1_f$2.err
  echo "sweep $1 f$2 rc=$?"
done
B="python bench.py --steps 5 --warmup 3 --reps 1 --no-e2e --no-cpu-baseline"
$B > $out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"vti|k_" -c 200 --csv --log-file $out/launches_C4.csv $B > $out/ncu_l.log 2>&1; echo "launches rc=$?"
for spec in "C4 32" "C2 32" "C3 32" "C5 32" "N1 32" "C2 64" "C3 64" "C5 64" "N1 64"; do
  set -- $spec
  B="python bench.py --config $1 --precision $2 --steps 4 --warmup 3 --reps 1 --no-e2e --no-cpu-baseline"
  rep=$out/prof_$1_f$2
  $B > $out/plain_$1_$2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:vti_step_kernel -s 3 -c 1 -o $rep $B > $out/ncu_$1_$2.log 2>&1; echo "ncu $1 f$2 rc=$?"
  ncu -i $rep.ncu-rep --page raw --csv > ${rep}_raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page details --csv > ${rep}_details.csv 2>/dev/null
  rm -f $rep.ncu-rep
done
du -sh $out
