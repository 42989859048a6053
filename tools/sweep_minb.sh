mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_counter.py -q -x > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
for m in 3 2 4; do
  CLGEN_CTR_MINB=$m timeout 400 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/sm_$m.log 2>&1
done
