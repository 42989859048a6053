"""C2 (uniform w = 50, n = 1e7, ~2.5e8 edges) through the counter stream's materialised path
(count pass, scan, replaying write pass, device radix sort into (u, v) order), device output."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1406_1215_b200 import api
w = np.full(10_000_000, 50.0)
ws = api.make_weight_sequence(w)
out = torch.empty((260_000_000, 2), dtype=torch.int32, device="cuda:0")
for rep in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    e = api.generate_range(ws, ws.sum_S, 0, w.size, 7 + rep, out=out)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print("C2 counter materialised:", int(e.shape[0]), "edges", round(dt * 1e3, 2), "ms", round(int(e.shape[0]) / dt / 1e9, 2), "G edges/s")
