echo "== parity: $(timeout 900 python -m pytest tests/test_fp64_gpu.py -m gpu -q 2>&1 | tail -1)"
run() { out=$(env $1 timeout 600 python bench.py --config $2 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline $3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['schedule'])" 2>&1); echo "$1 $2 $3 => $out"; }
for c in C2 C3 C5 N1; do run "" $c "--precision 64"; run "VTI_TY=16" $c "--precision 64"; done
