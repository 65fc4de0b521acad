"""Timeline of one cfg-5 rfd_gfi step (every launch's start / end on its
stream, profile mode: events around each launch) -> gpurun_out/timeline.txt"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

if len(sys.argv) > 1:
    rfd.load_library(sys.argv[1])
out = "gpurun_out/timeline.txt"
os.makedirs("gpurun_out", exist_ok=True)
if os.path.exists(out):
    os.remove(out)
p, x, F = make_config(5)
xd, Fd = torch.from_numpy(x).cuda(), torch.from_numpy(F).cuda()
o = torch.empty_like(Fd)
for _ in range(3):
    rfd.gfi(xd, p["eps"], p["lam"], p["m"], p["seed"], Fd, out=o)
torch.cuda.synchronize()
rfd.profile_enable(True)
rfd.profile_read()
os.environ["RFD_TIMELINE"] = out
rfd.gfi(xd, p["eps"], p["lam"], p["m"], p["seed"], Fd, out=o)
torch.cuda.synchronize()
rfd.profile_read()
print(open(out).read())
