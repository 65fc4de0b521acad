"""Top SASS instructions by warp-stall samples, with the stall-reason split.

    python tools/ncu_sass.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
keys = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[i_s] or 0) for r in data)
top = sorted(range(len(data)), key=lambda i: -float(data[i][i_s] or 0))[:N]
for i in sorted(top):
    r = data[i]
    split = {k[6:]: int(float(r[hdr.index(k)])) for k in keys
             if r[hdr.index(k)] not in ("0", "") and float(r[hdr.index(k)]) >= 0.1 * float(r[i_s] or 1)}
    print(f"{i:5d} {100 * float(r[i_s] or 0) / tot:5.1f}%  {r[1][:60]:60s} {split}")
