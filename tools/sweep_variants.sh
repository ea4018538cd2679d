# parity for each compiled variant (env-selected), then throughput per config
for v in "VTI_TY=32 VTI_RPT=1" "VTI_TY=32 VTI_RPT=2" "VTI_TY=16 VTI_RPT=1"; do
  echo "== parity $v: $(env $v timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x 2>&1 | tail -1)"
done
run() { out=$(env $1 timeout 600 python bench.py --config $2 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline $3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['schedule'])" 2>&1); echo "$1 $2 $3 => $out"; }
for c in C2 C3 C4 C5; do
  for v in "VTI_TY=32 VTI_RPT=1" "VTI_TY=32 VTI_RPT=2" "VTI_TY=16 VTI_RPT=1"; do run "$v" $c ""; done
done
run "VTI_TY=32 VTI_RPT=1" C2 "--zchunk 128"
run "VTI_TY=32 VTI_RPT=2" C2 "--zchunk 128"
