# class width x chunk size sweep of the counter sampler: lines "config eps chunk G-edges/s kernel-ms"
mkdir -p gpurun_out; rm -f gpurun_out/sweep_ec.log
for cfg in ${CONFIGS:-c3 c5}; do
  for eps in ${EPS:-0.0078125 0.03125 0.0625 0.125}; do
    for ch in ${CHUNKS:-4096 16384 65536}; do
      CLGEN_CTR_EPS=$eps CLGEN_CTR_CHUNK=$ch timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/sw.tmp 2>&1
      python -c "
import json
l=[x for x in open('gpurun_out/sw.tmp') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print('$cfg', $eps, $ch, d.get('value',0)/1e9, d.get('roofline',{}).get('kernel_ms'))" >> gpurun_out/sweep_ec.log
    done
  done
done
cat gpurun_out/sweep_ec.log
