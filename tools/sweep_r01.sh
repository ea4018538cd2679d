run() { out=$(env $1 timeout 600 python bench.py --config $2 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline $3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['schedule']['zchunk'])" 2>&1); echo "$1 $2 $3 => $out"; }
for promo in 256 128 none; do
  run VTI_P_PROMO=$promo C4 ""
  run VTI_P_PROMO=$promo C4 "--zchunk 1024"
  run VTI_P_PROMO=$promo C3 ""
  run VTI_P_PROMO=$promo C3 "--zchunk 512"
  run VTI_P_PROMO=$promo C2 ""
done
run VTI_P_PROMO=256 C4 "--zchunk 512"
run VTI_P_PROMO=256 C4 "--zchunk 64"
run VTI_P_PROMO=256 C2 "--zchunk 128"
run VTI_P_PROMO=256 C2 "--zchunk 512"
