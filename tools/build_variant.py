"""Build an A/B variant of librfd.so: the listed sources recompiled with extra
nvcc flags, every other object taken from the regular build.

    python tools/build_variant.py NAME "-DRFD_POLY_PAIRS=0" k_pass2_tc.cu [more.cu]
    -> abtest/NAME/librfd.so   (then: python tools/ab_time.py --lib abtest/NAME/librfd.so)
"""
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_00942_b200 import build as B  # noqa: E402

name, flags, srcs = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
B.build()
out = os.path.join(B.ROOT, "abtest", name)
os.makedirs(out, exist_ok=True)
objs = []
for o in sorted(glob.glob(os.path.join(B.OBJ, "*.o"))):
    base = os.path.basename(o)[:-2] + ".cu"
    if base in srcs:
        vo = os.path.join(out, os.path.basename(o))
        subprocess.run([B.nvcc()] + B.ARCH + B.FLAGS + flags + ["-c", os.path.join(B.CSRC, base), "-o", vo],
                       check=True)
        objs.append(vo)
    else:
        objs.append(o)
subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-cudart", "static", "-o", os.path.join(out, "librfd.so")] + objs,
               check=True)
print(os.path.join(out, "librfd.so"))
