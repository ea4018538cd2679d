echo "== parity: $(timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fp64_gpu.py tests/test_n4_gpu.py -m gpu -q -x 2>&1 | tail -1)"
run() { out=$(env $1 timeout 600 python bench.py --config $2 --steps 200 --warmup 10 --no-e2e --no-cpu-baseline $3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])" 2>&1); echo "$1 $2 $3 => $out"; }
for i in 1 2; do for v in "VTI_PDL=1" "VTI_PDL=0"; do run "$v" C2 ""; done; done
for v in "VTI_PDL=1" "VTI_PDL=0"; do run "$v" N1 ""; run "$v" C2 "--precision 64"; done
