#!/bin/bash
for h in 16 32 64 128; do
  echo "heavy=$h c3: $(CLGEN_CTR_HEAVY=$h python tools/ref_info.py c3 1e8 counter | tail -1) | c4n1e8: $(CLGEN_CTR_HEAVY=$h python tools/ref_info.py c4 1e8 counter | tail -1)"
done
