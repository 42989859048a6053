# counter-stream law/determinism tests, then A/B of kernel shapes at C4 shape n=2e8 (each line one bench run)
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
timeout 1200 python -m pytest tests/test_gpu_counter.py tests/test_gpu_law.py -q -x -k "not fullsize and not c4_full" > gpurun_out/t_ctr.log 2>&1; echo rc=$? >> gpurun_out/t_ctr.log
bash tools/ab_blk.sh "${@}"
cat gpurun_out/ab.log
tail -3 gpurun_out/t_ctr.log
