#!/bin/bash
# Quick variant sweep: tools/sweep.sh "<bench args>" "ENV=V ENV2=V2" "ENV=V" ...  (one bench line per variant)
set -u
args=$1; shift
mkdir -p gpurun_out
i=0
for V in "$@"; do
  i=$((i+1))
  env $V timeout 600 python bench.py $args --no-e2e --no-cpu-baseline > gpurun_out/sw_$i.log 2>&1
  echo "$i [$V] $(grep '^{' gpurun_out/sw_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,2), round(d["ms_per_step"],1))' 2>/dev/null)" >> gpurun_out/sweep.txt
done
