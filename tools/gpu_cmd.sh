timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tall.log 2>&1; echo rc=$? >> gpurun_out/tall.log
for c in c5 c3 c4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/e2e_$c.log 2>&1; done
