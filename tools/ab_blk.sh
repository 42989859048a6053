# A/B of counter-sampler variants at C4 shape: each line = one bench run (sampler kernel ms in roofline.kernel_ms)
mkdir -p gpurun_out
N=${AB_N:-200000000}
for v in "${@}"; do
  env $v timeout 600 python bench.py --config c4 --num-vertices $N --no-cpu-baseline --no-e2e --steps 3 --warmup 2 > gpurun_out/ab.tmp 2>&1
  python -c "
import json,sys
l=[x for x in open('gpurun_out/ab.tmp') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print('$v', d.get('value',0)/1e9 if d else open('gpurun_out/ab.tmp').read()[-300:], d.get('roofline',{}).get('kernel_ms'))" >> gpurun_out/ab.log
done
