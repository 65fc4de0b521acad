"""SASS opcode histogram per kernel of the built library (no GPU needed).

    python tools/sass_histogram.py [lib/librfd.so] > profiles/r02_sass_histogram.txt

Per kernel: total instructions and the counts of the opcodes that evidence
the design (tcgen05 MMA: UTCHMMA / UTCHMMA.2CTA, TMEM: LDTM / STTM, TMA /
bulk copies: UBLKCP / UTMALDG, fp64 tensor: DMMA, packed FP32: FFMA2 /
FMUL2, the sin/cos pipe: MUFU.SIN / MUFU.COS, fp16 splits: F2FP).
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2302_00942_b200", "lib", "librfd.so")
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["UTCHMMA", "UTCHMMA.2CTA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "LDGSTS", "DMMA",
        "FFMA2", "FMUL2", "FFMA", "MUFU.SIN", "MUFU.COS", "MUFU.EX2", "MUFU.LG2", "F2FP", "FHFMA",
        "SYNCS", "LDS", "STS", "LDG", "STG", "SHFL", "ATOMG", "REDG"]
funcs = re.split(r"\n\s*Function : ", txt)[1:]
rows = []
for f in funcs:
    name = f.split("\n")[0].strip()
    ops = collections.Counter()
    for line in f.split("\n"):
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+(?:\.[A-Z0-9_]+)*)", line)
        if m:
            op = m.group(1)
            ops[op] += 1
    total = sum(ops.values())
    agg = collections.Counter()
    for op, c in ops.items():
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                agg[k] += c
        if op.startswith("UTCHMMA") and "2CTA" in op:
            agg["UTCHMMA.2CTA"] += c
    dem = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()
    dem = dem.replace("(anonymous namespace)::", "").replace("void ", "")
    depth, cut = 0, len(dem)
    for i, ch in enumerate(dem):  # strip the argument list (after the template arguments)
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif ch == "(" and depth == 0:
            cut = i
            break
    short = dem[:cut].replace("rfd::", "")
    rows.append((short, total, agg))
print("# SASS opcode histogram per kernel (cuobjdump -sass of %s)" % os.path.relpath(lib, ROOT))
print("# columns: total instructions, then counts of: " + ", ".join(KEYS))
for short, total, agg in sorted(rows):
    parts = ["%s=%d" % (k, agg[k]) for k in KEYS if agg[k]]
    print("%-44s %6d  %s" % (short[:44], total, " ".join(parts)))
