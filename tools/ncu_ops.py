"""Per-opcode executed-instruction counts and stall-sample shares of one
kernel in an ncu report (SASS source page).

    python tools/ncu_ops.py report.ncu-rep KERNEL_REGEX [units] [N]
(units: divide the thread-instruction counts by this, e.g. the point count)
"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, kre = sys.argv[1], sys.argv[2]
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
N = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = {k: i for i, k in enumerate(rows[1])}
ops, smp = Counter(), Counter()
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    ie = int(r[hdr["Instructions Executed"]].replace(",", "") or 0)
    t = r[hdr["Source"]].strip().split()
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ops[op] += ie
    smp[op] += int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
tot, ts = sum(ops.values()), sum(smp.values()) or 1
print("warp instructions %d, thread instructions per unit %.1f" % (tot, tot * 32 / units))
for k, v in ops.most_common(N):
    print("%-9s %11d %5.1f%%  per unit %7.1f  stall samples %5.1f%%" % (k, v, 100 * v / tot, v * 32 / units,
                                                                     100 * smp[k] / ts))
