#!/bin/bash
for eps in 0.03125 0.0625 0.125 0.25; do
  echo "eps=$eps $(CLGEN_CTR_EPS=$eps python tools/ref_info.py c4 1e8 counter | tail -1) | c3: $(CLGEN_CTR_EPS=$eps python tools/ref_info.py c3 1e8 counter | tail -1) | c5: $(CLGEN_CTR_EPS=$eps python tools/ref_info.py c5 1e7 counter | tail -1)"
done
