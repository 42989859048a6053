"""Time the reference-stream fold on a workload (kernel ms)."""
import sys, time
sys.path.insert(0, '.')
from paper_1406_1215_b200 import api
import inputs as workloads
name = sys.argv[1]; n = int(float(sys.argv[2])) if len(sys.argv) > 2 else None
mode = sys.argv[3] if len(sys.argv) > 3 else "reference"
w = workloads.make(name, n)
ws = api.make_weight_sequence(w)
for rep in range(2):
    r = api.stream_range(ws, ws.sum_S, 0, w.size, 7, mode=mode, track_shift=6)
    print(mode, "edges", r.count, "flagged", r.flagged, "kernel ms", round(ws.device.last_kernel_ms(), 2))
