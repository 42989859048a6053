#!/bin/bash
# Short final pass after the last kernel change: bench lines, launch list at C4, full capture at n = 2e8.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
for c in c3 c5; do timeout 300 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; done
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum --clock-control none --csv \
    --log-file gpurun_out/c4_bench_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/c4_ncu_launches.log 2>&1
NCU_N=200000000 NCU_OUT=blk_final bash tools/ncu_blk_full.sh
