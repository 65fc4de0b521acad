"""Per-kernel times of a cfg plan + integrate with a given librfd.so (A/B of
kernel variants on the same box).

    python tools/ab_time.py --lib path/to/librfd.so [--cfg 5] [--reps 10]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=rfd.LIB_PATH)
ap.add_argument("--cfg", type=int, default=5)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--integrates", type=int, default=1)
a = ap.parse_args()
rfd.load_library(a.lib)
p, x, F = make_config(a.cfg)
if a.cfg == 3:
    F = F[0]
xd, Fd = torch.from_numpy(x).cuda(), torch.from_numpy(F).cuda()
od = torch.empty_like(Fd)
for _ in range(3):
    pl = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    pl.integrate(Fd, out=od)
    pl.close()
torch.cuda.synchronize()
rfd.profile_enable(True)
rfd.profile_read()
for _ in range(a.reps):
    pl = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    for _ in range(a.integrates):
        pl.integrate(Fd, out=od)
    pl.close()
prof = rfd.profile_read()
print(json.dumps({"lib": a.lib, "cfg": a.cfg,
                  "ms": {k: v[1] / v[0] for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])}}))
