# ncu evidence for the class-pair block sampler (run each only after the plain command exited 0)
mkdir -p gpurun_out
N=${NCU_N:-200000000}
timeout 600 python bench.py --config c4 --num-vertices $N --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > gpurun_out/ncu_pre.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum --clock-control none --csv \
    --log-file gpurun_out/blk_launches.csv python bench.py --config c4 --num-vertices $N --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:blk_kernel -c 1 \
    -o gpurun_out/blk_full python bench.py --config c4 --num-vertices $N --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1
ls -la gpurun_out
