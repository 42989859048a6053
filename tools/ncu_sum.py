"""Summarise an ncu --csv metrics log (one row per kernel/metric)."""
import collections
import csv
import sys

for fn in sys.argv[1:]:
    rows = list(csv.reader(open(fn)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = (d["ID"], d["Kernel Name"].split("(")[0][:48])
        agg.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    print("==", fn)
    for k, v in agg.items():
        t = v.get("gpu__time_duration.sum", 0) / 1e6
        ins = v.get("smsp__inst_executed.sum", 0)
        th = v.get("smsp__thread_inst_executed.sum", 0)
        print(f"{k[0]:>3} {k[1]:48s} {t:9.2f} ms  inst {ins:.4g}  lanes/inst {th / max(ins, 1):.1f}  "
              f"dramW {v.get('dram__bytes_write.sum', 0) / 1e9:.1f} GB  dramR {v.get('dram__bytes_read.sum', 0) / 1e9:.1f} GB")
