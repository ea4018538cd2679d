#!/bin/bash
# Throughput sweep over env-selected kernel variants / schedules (run on a B200):
#   bash tools/sweep.sh "VTI_TY=32 VTI_WP=1|C2|" "VTI_TY=30 VTI_WP=1|C4|--zchunk 512" ...
# Each argument is "ENV|CONFIG|EXTRA bench.py args". Env knobs (read at vti_create):
#   VTI_TY (32|30|16|15|14|10|8), VTI_WP (1|0), VTI_RPT (1|2), VTI_PX (4|2), VTI_ALIGN (1|0),
#   VTI_LAYOUT (zyx|yzx), VTI_P_PROMO (none|64|128|256), VTI_SAT (CTAs that saturate HBM),
#   VTI_MAXGRID (CTA cap), VTI_SMALL / VTI_PDL (small-grid kernel) -- see README.md.
for spec in "$@"; do
  IFS='|' read -r envs cfg extra <<< "$spec"
  out=$(env $envs timeout 600 python bench.py --config "$cfg" --steps 30 --warmup 3 --no-e2e --no-cpu-baseline $extra 2>&1 | tail -1 |
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['schedule'])" 2>&1)
  echo "$envs $cfg $extra => $out"
done
