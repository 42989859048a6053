#!/bin/bash
# Round-2 measurement pass on the GPU box (run via gpurun). Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
bash tools/round_measure.sh
# launch list at full C4 (cold-cache, serialised: shares only), then one full capture
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum --clock-control none --csv \
    --log-file gpurun_out/c4_bench_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/c4_ncu_launches.log 2>&1
NCU_N=200000000 NCU_OUT=blk_final bash tools/ncu_blk_full.sh
ls -la gpurun_out
