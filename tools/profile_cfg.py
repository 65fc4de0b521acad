"""Per-kernel device time of rfd_integrate at one config (profile API).

    python tools/profile_cfg.py CFG [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

cfg = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p, x, F = make_config(cfg)
if cfg == 3:
    F = F[0]
xd, Fd = torch.from_numpy(x).cuda(), torch.from_numpy(F).cuda()
plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
for _ in range(5):
    plan.integrate(Fd)
torch.cuda.synchronize()
rfd.profile_enable(True)
rfd.profile_read()
for _ in range(reps):
    plan.integrate(Fd)
prof = rfd.profile_read()
rfd.profile_enable(False)
tot = 0.0
for name, (cnt, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    print("%-22s %5d launches  %8.2f us/launch" % (name, cnt, 1e3 * ms / cnt))
    tot += ms
print("total per integrate: %.2f us" % (1e3 * tot / reps))
