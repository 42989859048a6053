# chunk-size sweep of the counter sampler per config: lines "config chunk shape G-edges/s kernel-ms"
mkdir -p gpurun_out; rm -f gpurun_out/sweep_chunk.log
for cfg in ${CONFIGS:-c3 c5}; do
  for ch in ${CHUNKS:-2048 4096 8192 16384 32768 65536 131072}; do
    for sh in ${SHAPES:-1 2}; do
      CLGEN_CTR_CHUNK=$ch CLGEN_BLK_SHAPE=$sh timeout 600 python bench.py --config $cfg ${EXTRA:-} --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/sw.tmp 2>&1
      python -c "
import json
l=[x for x in open('gpurun_out/sw.tmp') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print('$cfg', $ch, $sh, d.get('value',0)/1e9, d.get('roofline',{}).get('kernel_ms'))" >> gpurun_out/sweep_chunk.log
    done
  done
done
cat gpurun_out/sweep_chunk.log
