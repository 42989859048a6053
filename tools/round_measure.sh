#!/bin/bash
# Full measurement pass on the GPU box (run via gpurun). Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
for c in c1 c2; do timeout 300 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; done
for c in c3 c5; do timeout 300 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; done
timeout 600 python bench.py --mode reference --no-e2e --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_c4_refstream.log 2>&1
