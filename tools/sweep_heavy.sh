mkdir -p gpurun_out
for h in 64 96 128 192; do
  CLGEN_CTR_HEAVY=$h timeout 400 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/sh_$h.log 2>&1
done
