run() { env $1 timeout 600 python bench.py --config C2 --steps 200 --warmup 10 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['roofline']['frac'], d['clocks'])"; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
for i in 1 2 3; do run "VTI_RPT=1"; run "VTI_RPT=2 VTI_WP=0"; done
