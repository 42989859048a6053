bash tools/round_measure.sh
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv \
    --log-file gpurun_out/c4_bench_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/c4_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ctr_warp_kernel -c 1 \
    -o gpurun_out/c4_ctr_warp_full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/c4_ncu_full.log 2>&1
