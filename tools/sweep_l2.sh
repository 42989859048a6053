#!/bin/bash
for g in 0 32 64; do for p in 0 64; do
  echo "fetch=$g persistMB=$p $(CLGEN_L2_FETCH=$g CLGEN_L2_PERSIST_MB=$p python tools/ref_info.py c4 1e8 reference | tail -1) | $(CLGEN_L2_FETCH=$g CLGEN_L2_PERSIST_MB=$p python tools/ref_info.py c4 1e8 counter | tail -1)"
done; done
