"""One cfg-N plan creation (Gram + core), errors from diagnostic modes ignored: an ncu target.

    RFD_GRAM_MODE=2 python tools/gram_once.py [cfg]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

p, x, F = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
xd = torch.from_numpy(x).cuda()
try:
    rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"]).close()
except rfd.RFDError as e:
    print("plan:", e)
torch.cuda.synchronize()
print("ok")
