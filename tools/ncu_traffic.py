"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
kernels in an `ncu --set full` report, keyed by the library's launch-scope
names, as JSON (read by bench.py for roofline.traffic).

    python tools/ncu_traffic.py gpurun_out/full.ncu-rep [more.ncu-rep ...] > profiles/traffic.json
"""
import csv
import io
import json
import re
import subprocess
import sys

SCOPES = [(r"gram_pair_kernel|gram_tc_kernel", "rfd_gram_tc"), (r"pass1_tc", "rfd_pass1_tc"),
          (r"pass2_tc", "rfd_pass2_tc"), (r"dgemm_kernel", "rfd_core_dgemm"),
          (r"nufft_spread", "rfd_nufft_spread")]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

acc = {}
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    k, r, w = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    for row in rows[2:]:
        name = next((s for pat, s in SCOPES if re.search(pat, row[k])), None)
        if name is None:
            continue
        b = float(row[r]) * UNIT[units[r]] + float(row[w]) * UNIT[units[w]]
        e = acc.setdefault(name, {"sum": 0.0, "launches": 0, "report": rep.split("/")[-1]})
        e["sum"] += b
        e["launches"] += 1
print(json.dumps({n: {"bytes_per_launch": e["sum"] / e["launches"], "launches": e["launches"],
                      "report": e["report"]} for n, e in acc.items()}, indent=1))
