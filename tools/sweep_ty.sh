run() { out=$(env $1 timeout 600 python bench.py --config $2 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline $3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['schedule'])" 2>&1); echo "$1 $2 $3 => $out"; }
for ty in 32 16; do
  for c in C2 C3 C4 C5; do run VTI_TY=$ty $c ""; done
  run VTI_TY=$ty C2 "--zchunk 128"
  run VTI_TY=$ty C2 "--zchunk 512"
  run VTI_TY=$ty C4 "--zchunk 1024"
  run VTI_TY=$ty C3 "--zchunk 512"
done
