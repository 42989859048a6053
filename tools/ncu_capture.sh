#!/bin/bash
# Usage (on the GPU box, via gpurun): tools/ncu_capture.sh <tag> <kernel-regex> <bench args...>
# 1) runs the bench command plainly (must exit 0), 2) the launch list with
# per-launch device time, 3) one `--set full` capture of the top kernel.
set -u
tag=$1; kre=$2; shift 2
mkdir -p gpurun_out
python bench.py "$@" --no-e2e --no-cpu-baseline > gpurun_out/${tag}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv python bench.py "$@" --no-e2e --no-cpu-baseline \
    > gpurun_out/${tag}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:${kre} -s ${NCU_SKIP:-1} -c 1 \
    -o gpurun_out/${tag} python bench.py "$@" --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_full.log 2>&1
echo done
