# counter-stream GPU tests + C4/C3 bench lines (used while tuning the counter kernels)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_counter.py -q -x > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
for c in c4 c3; do
  timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/q_$c.log 2>&1
done
if [ -n "${EXTRA_ENV:-}" ]; then
  env $EXTRA_ENV timeout 400 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/q_c4x.log 2>&1
fi
