mkdir -p gpurun_out
{
for eps in 0.00390625 0.0078125 0.015625; do
  echo "eps=$eps c4: $(CLGEN_CTR_EPS=$eps timeout 120 python tools/ref_info.py c4 2e8 counter | tail -1) | c3: $(CLGEN_CTR_EPS=$eps timeout 120 python tools/ref_info.py c3 1e8 counter | tail -1)"
done
for h in 256 512; do
  echo "heavy=$h c4: $(CLGEN_CTR_HEAVY=$h timeout 120 python tools/ref_info.py c4 2e8 counter | tail -1) | c3: $(CLGEN_CTR_HEAVY=$h timeout 120 python tools/ref_info.py c3 1e8 counter | tail -1)"
done
} > gpurun_out/sweep_final.log 2>&1
