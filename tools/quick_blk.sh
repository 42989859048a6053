# counter-stream (class-pair block sampler) GPU tests + bench lines
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_counter.py -q -x ${PYTEST_K:-} > gpurun_out/t_ctr.log 2>&1; echo rc=$? >> gpurun_out/t_ctr.log
for c in ${CONFIGS:-c4 c3 c5}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/q_$c.log 2>&1
done
