#!/bin/bash
# A/B of library builds on the GPU box:
#   tools/ab.sh "<bench args>" lib1.so[:ENV=V[,ENV2=V2]] lib2.so ...
# Plain bench lines (alternating, 2 passes) then an ncu instruction/time count
# of the sampler kernels per variant.  Outputs in gpurun_out/ab_*.
set -u
args=$1; shift
mkdir -p gpurun_out
tagof() { local L=${1%%:*}; local E=""; [[ "$1" == *:* ]] && E=${1#*:}; echo "$(basename $L .so)${E:+_${E//[=,]/_}}"; }
envof() { [[ "$1" == *:* ]] && echo "${1#*:}" | tr ',' ' '; }
for pass in 1 2; do
  for V in "$@"; do
    L=${V%%:*}; t=$(tagof "$V")
    env CLGEN_LIB=$PWD/$L $(envof "$V") timeout 600 python bench.py $args --no-e2e --no-cpu-baseline > gpurun_out/ab_${t}_$pass.log 2>&1
  done
done
for V in "$@"; do
  L=${V%%:*}; t=$(tagof "$V")
  env CLGEN_LIB=$PWD/$L $(envof "$V") timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,dram__bytes_write.sum,dram__bytes_read.sum \
    --clock-control none -k regex:ctr_ --csv --log-file gpurun_out/ab_${t}_ncu.csv \
    python bench.py $args --no-e2e --no-cpu-baseline --steps 1 --warmup 0 > /dev/null 2>&1
done
echo done
