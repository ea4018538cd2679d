echo "== parity (defaults): $(timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fp64_gpu.py -m gpu -q -x 2>&1 | tail -1)"
echo "== parity TY30: $(VTI_TY=30 VTI_WP=1 timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k 'random_state or c1_full or local_group_short or fullsize' 2>&1 | tail -1)"
run() { out=$(env $1 timeout 600 python bench.py --config $2 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline $3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['schedule'])" 2>&1); echo "$1 $2 $3 => $out"; }
for c in C2 C3 C4; do for v in "VTI_TY=32 VTI_WP=1" "VTI_TY=30 VTI_WP=1"; do run "$v" $c ""; done; done
run "" C5 ""; run "" N1 ""
for v in "VTI_WP=1" "VTI_WP=0"; do run "$v" N1 "--precision 64"; run "$v" C5 "--precision 64"; done
