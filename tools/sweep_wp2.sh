echo "== parity: $(timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fp64_gpu.py tests/test_n4_gpu.py -m gpu -q -x 2>&1 | tail -1)"
run() { out=$(env $1 timeout 600 python bench.py --config $2 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline $3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'])" 2>&1); echo "$1 $2 $3 => $out"; }
for c in C2 C3 C4 C5 N1; do for v in "VTI_WP=1 VTI_RPT=1" "VTI_WP=0 VTI_RPT=1"; do run "$v" $c ""; done; done
run "VTI_WP=1" C2 "--precision 64"
run "VTI_WP=0" C2 "--precision 64"
