# class-width sweep of the counter sampler per config: lines "config eps G-edges/s kernel-ms"
mkdir -p gpurun_out; rm -f gpurun_out/sweep_eps.log
for cfg in ${CONFIGS:-c3 c5}; do
  for eps in ${EPS:-0.0078125 0.015625 0.03125 0.0625 0.125}; do
      CLGEN_CTR_EPS=$eps CLGEN_BLK_SHAPE=${SHAPE:-1} timeout 600 python bench.py --config $cfg ${EXTRA:-} --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/sw.tmp 2>&1
      python -c "
import json
l=[x for x in open('gpurun_out/sw.tmp') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print('$cfg', $eps, d.get('value',0)/1e9, d.get('roofline',{}).get('kernel_ms'))" >> gpurun_out/sweep_eps.log
  done
done
cat gpurun_out/sweep_eps.log
