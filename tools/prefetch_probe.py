"""Does the prefetched weight copy overlap the generation?  Wall-clock probes around the calls."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1406_1215_b200 import api
import inputs
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 200_000_000
w = inputs.make("c4", n)
pin = torch.from_numpy(w).pin_memory()
dev = api.Device(0)
ring = torch.empty((1 << 28, 2), dtype=torch.int32, device="cuda:0")
def gen():
    S = dev.blocked_sum()
    ws = api.WeightSequence(w, S, None, dev)
    return api.stream_range(ws, S, 0, n, 7, mode="counter", track_shift=6, ring=ring).count
for mode in ("serial", "prefetch", "serial", "prefetch"):
    dev.set_weights(pin); gen()
    torch.cuda.synchronize()
    t = []
    for _ in range(3):
        t0 = time.perf_counter()
        dev.set_weights(pin)
        t1 = time.perf_counter()
        if mode == "prefetch":
            dev.prefetch_weights(pin)
        t2 = time.perf_counter()
        gen()
        t3 = time.perf_counter()
        t.append((round((t1 - t0) * 1e3, 1), round((t2 - t1) * 1e3, 1), round((t3 - t2) * 1e3, 1)))
    print(mode, "set_weights / prefetch call / generate (ms):", t)
