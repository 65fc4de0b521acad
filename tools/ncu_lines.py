"""Warp-stall samples aggregated per CUDA source line (ncu --print-source cuda,sass).

    python tools/ncu_lines.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
per = defaultdict(float)
text = {}
hdr = None
cur_file = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    try:
        v = float(r[hdr["Warp Stall Sampling (All Samples)"]].replace(",", "") or 0)
    except ValueError:
        continue
    key = (cur_file, r[0])
    per[key] += v
    text[key] = r[1]
tot = sum(per.values()) or 1.0
for k, v in sorted(per.items(), key=lambda kv: -kv[1])[:N]:
    print("%5.1f%%  %s:%s  %s" % (100 * v / tot, k[0], k[1], text[k].strip()[:100]))
