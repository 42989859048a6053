#!/bin/bash
for r in 1 4 8 16; do
  for c in c1 c2; do
    v=$(CLGEN_REFILL_MIN=$r timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['value']/1e9,2), round(d['ms_per_step'],3), [round(x['max_over_mean'],2) for x in d['load_balance']['per_launch_warp_busy']])")
    echo "refill_min=$r $c $v"
  done
done
