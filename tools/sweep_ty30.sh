for v in "VTI_TY=30 VTI_WP=1" ; do echo "== parity $v: $(env $v timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k 'random_state or c1_full or local_group_short' 2>&1 | tail -1)"; done
run() { out=$(env $1 timeout 600 python bench.py --config $2 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline $3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['schedule'])" 2>&1); echo "$1 $2 $3 => $out"; }
for c in C5 N1; do for v in "" "VTI_TY=30 VTI_WP=1"; do run "$v" $c ""; done; done
