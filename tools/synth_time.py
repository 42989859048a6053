"""Time clgen_dev_synth_powerlaw on the C4 recipe (default n = 1e9) and compare
the array with the host synthesiser's (inputs.make('c4')) bit for bit.
    python tools/synth_time.py [n] [--no-check]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1406_1215_b200 import api  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else 1_000_000_000
dev = api.default_device(0)
api.synth_powerlaw_device(1 << 20, 2.5, 1.0, 1000.0, 1, dev)  # warm-up: jump matrices, module load
out = {"n": n}
for label, kw in (("draws_only", dict(sort=False)), ("draws_sort_scale", dict(sort=True, target_mean=500.0))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    w, resolved = api.synth_powerlaw_device(n, 2.5, 1.0, 1000.0, 1, dev, **kw)
    torch.cuda.synchronize()
    out[label + "_s"] = round(time.perf_counter() - t0, 4)
    out["host_resolved"] = resolved
    if label == "draws_only":
        del w
        torch.cuda.empty_cache()
if "--no-check" not in sys.argv:
    import inputs
    t0 = time.perf_counter()
    want = inputs.make("c4", n)
    out["host_synth_s"] = round(time.perf_counter() - t0, 2)
    got = w.cpu().numpy()
    out["bit_identical"] = bool(np.array_equal(got.view(np.uint64), want.view(np.uint64)))
print(json.dumps(out))
