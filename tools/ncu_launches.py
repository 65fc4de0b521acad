"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel launches, total device time and share (cold-cache, serialised)."""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "s": 1e3, "second": 1e3}


def summarise(path, skip_first=0):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1 + skip_first:]:
        name = r[ki].split("(")[0].split("::")[-1].split("<")[0]
        v = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    out = ["%-28s %7s %12s %7s" % ("kernel", "launches", "total ms", "share")]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append("%-28s %7d %12.3f %6.1f%%" % (k, v[0], v[1], 100 * v[1] / tot))
    out.append("%-28s %7d %12.3f" % ("TOTAL", sum(v[0] for v in agg.values()), tot))
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
