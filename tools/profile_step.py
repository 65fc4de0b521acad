"""One cfg-5 plan + integrate through the C ABI: a short command for ncu.

    python tools/profile_step.py [--cfg 5] [--reps 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=5)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
p, x, F = make_config(a.cfg)
xd, Fd = torch.from_numpy(x).cuda(), torch.from_numpy(F).cuda()
for _ in range(a.reps):
    plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    out = plan.integrate(Fd)
    plan.close()
torch.cuda.synchronize()
print("ok", float(out.abs().max()))
