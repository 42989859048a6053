"""Summarise one ncu report of a kernel: headline metrics, stall reasons per issue, pipe use, and
per-SASS-region instruction counts per loop iteration.
usage: python tools/ncu_report.py REPORT.ncu-rep [edges]"""
import csv, io, subprocess, sys

def page(rep, name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))

rep = sys.argv[1]
edges = float(sys.argv[2]) if len(sys.argv) > 2 else None
rows = page(rep, "details")
h = rows[0]
want = ('Duration', 'Executed Ipc Active', 'Issue Slots Busy', 'Executed Instructions', 'Registers Per Thread',
        'Eligible Warps Per Scheduler', 'No Eligible', 'Warp Cycles Per Issued Instruction',
        'Avg. Active Threads Per Warp', 'Avg. Not Predicated Off Threads Per Warp', 'Achieved Occupancy',
        'DRAM Throughput', 'Memory Throughput', 'Grid Size', 'Theoretical Occupancy')
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get('Metric Name') in want:
        print(f"{d['Section Name'][:24]:24s} | {d['Metric Name']} | {d['Metric Value']} {d['Metric Unit']}")
rows = page(rep, "raw")
d = dict(zip(rows[0], rows[2] if len(rows) > 2 else rows[1]))
print("stall cycles per issued instruction:")
st = []
for k in d:
    if k.startswith('smsp__average_warps_issue_stalled') and k.endswith('per_issue_active.ratio'):
        st.append((float(d[k]), k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
print("  " + ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True) if v > 0.05))
print("pipes (% of peak sustained active):")
for p in ('alu', 'fma', 'fp64', 'xu', 'lsu', 'adu', 'cbu', 'uniform'):
    print(f"  {p} {d.get(f'sm__inst_executed_pipe_{p}.avg.pct_of_peak_sustained_active')}", end="")
print()
for k in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum'):
    v = d.get(k)
    if v:
        x = float(v.replace(',', ''))
        print(f"  {k} {x:.4g}" + (f" ({x / edges:.3f} per edge)" if edges else ""))
