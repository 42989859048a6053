"""Print the counter plan (classes, hubs, units, heavy units) for a workload."""
import sys, time
sys.path.insert(0, '.')
import torch
from paper_1406_1215_b200 import api
import inputs as workloads
name = sys.argv[1]; n = int(float(sys.argv[2])) if len(sys.argv) > 2 else None
w = workloads.make(name, n)
ws = api.make_weight_sequence(w)
for rep in range(2):
    t = time.time()
    r = api.stream_range(ws, ws.sum_S, 0, w.size, 7, mode="counter")
    print("edges", r.count, "kernel ms", ws.device.last_kernel_ms(), "wall", time.time() - t)
print(ws.device.counter_plan_info())
