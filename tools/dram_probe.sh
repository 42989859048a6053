# bench line + ncu DRAM bytes / time of blk_kernel at C4 shape n = 2e8 (one variant = the current build)
mkdir -p gpurun_out
N=${NCU_N:-200000000}
timeout 600 python bench.py --config c4 --num-vertices $N --no-cpu-baseline --no-e2e --steps 3 --warmup 2 2>&1 | grep "^{" | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('bench', d['value']/1e9, d['ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum --clock-control none --csv -k regex:blk_kernel \
    --log-file gpurun_out/dram_probe.csv python bench.py --config c4 --num-vertices $N --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/dram_probe.log 2>&1
python tools/ncu_sum.py gpurun_out/dram_probe.csv | tail -2
