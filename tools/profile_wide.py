"""Per-kernel device time of rfd_integrate on cfg-5 points with a d-column
synthetic field (multi-column path, NEXT-2).

    python tools/profile_wide.py D [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

d = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
p, x, _ = make_config(5)
xd = torch.from_numpy(x).cuda()
Fd = torch.randn((p["n"], d), device="cuda", generator=torch.Generator("cuda").manual_seed(1))
plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
for _ in range(3):
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
    print("%-22s %5d launches  %8.3f ms/launch  %8.3f ms/integrate" % (name, cnt, ms / cnt, ms / reps))
    tot += ms
print("d=%d total per integrate: %.3f ms" % (d, tot / reps))
