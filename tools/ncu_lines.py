"""Per-source-line instruction / stall attribution from an ncu report.

usage: python tools/ncu_lines.py REPORT.ncu-rep [per_unit_divisor] [top]
Reads `ncu -i REPORT --page source --csv --print-source cuda,sass` and sums
warp-level instructions executed and stall samples per CUDA source line.
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    f = None
    hdr = None
    agg = {}
    cur = None
    for x in rows:
        if not x:
            continue
        if x[0] == "File Path":
            f = x[1].rsplit("/", 1)[-1]
            continue
        if x[0] == "Line No":
            hdr = x
            ie = hdr.index("Instructions Executed")
            iw = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or x[0] == "Function Name":
            continue
        if x[0]:
            cur = (f, int(x[0]), x[1].strip()[:70])
            continue
        try:
            e = float(x[ie] or 0)
            w = float(x[iw] or 0)
        except (ValueError, IndexError):
            continue
        a = agg.setdefault(cur, [0.0, 0.0])
        a[0] += e
        a[1] += w
    te = sum(v[0] for v in agg.values())
    tw = sum(v[1] for v in agg.values())
    print(f"total instr {te:.4g} ({te / div:.1f} per unit), stall samples {tw:.0f}")
    for k, v in sorted(agg.items(), key=lambda t: -t[1][0])[:top]:
        print(f"{v[0] / div:8.2f} {100 * v[1] / max(tw, 1):5.1f}%  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()
