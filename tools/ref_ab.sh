# reference-stream tests + C1/C2 bench lines with and without the heavy phase
mkdir -p gpurun_out; rm -f gpurun_out/ref_ab.log
timeout 1500 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_gates.py -q -x > gpurun_out/t_ref.log 2>&1; echo rc=$? >> gpurun_out/t_ref.log
for h in 1 0; do for cfg in c1 c2; do
  CLGEN_REF_HEAVY=$h timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > gpurun_out/r.tmp 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/r.tmp') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
lb=d.get('load_balance',{}).get('per_launch_warp_busy',[{}])
print('heavy=$h', '$cfg', d.get('value',0)/1e9, d.get('ms_per_step'), d.get('roofline',{}).get('kernel_ms'), [ (x.get('max_over_mean'), x.get('max_ms')) for x in lb])" >> gpurun_out/ref_ab.log
done; done
cat gpurun_out/ref_ab.log; tail -3 gpurun_out/t_ref.log
