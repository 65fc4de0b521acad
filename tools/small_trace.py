"""One cfg's integrate with RFD_SMALL_TRACE=1 (phase timestamps on stderr)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p, x, F = make_config(cfg)
if cfg == 3:
    F = F[0]
plan = rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
Fd = torch.from_numpy(np.ascontiguousarray(F)).cuda()
od = torch.empty_like(Fd)
for _ in range(6):
    plan.integrate(Fd, out=od)
torch.cuda.synchronize()
