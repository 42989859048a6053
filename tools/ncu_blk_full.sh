# one full ncu capture of the counter sampler at C4 shape (n = NCU_N)
mkdir -p gpurun_out
N=${NCU_N:-200000000}
timeout 600 python bench.py --config c4 --num-vertices $N --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > gpurun_out/ncu_pre.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:blk_kernel -c 1 \
    -o gpurun_out/${NCU_OUT:-blk_full} -f python bench.py --config c4 --num-vertices $N --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1
