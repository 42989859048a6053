#!/bin/bash
for eps in 0.125 0.0625 0.03125; do for wm in 2 3 4; do
  r=$(CLGEN_CTR_EPS=$eps CLGEN_WARP_MINB=$wm python tools/ctr_info.py c4 1e8 2>&1 | grep "kernel ms" | tail -1)
  echo "eps=$eps wminb=$wm $r"
done; done
for h in 32 128; do r=$(CLGEN_CTR_HEAVY=$h python tools/ctr_info.py c4 1e8 2>&1 | grep "kernel ms" | tail -1); echo "heavy=$h $r"; done
for h in 16 32 64; do r=$(CLGEN_CTR_HEAVY=$h python tools/ctr_info.py c3 1e8 2>&1 | grep "kernel ms" | tail -1); echo "c3 heavy=$h $r"; done
