"""One cfg-5-points integrate with a d-column field (trace target).

    RFD_P2_TRACE=1 python tools/trace_wide.py D
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

d = int(sys.argv[1])
p, x, _ = make_config(5)
xd = torch.from_numpy(x).cuda()
Fd = torch.randn((p["n"], d), device="cuda", generator=torch.Generator("cuda").manual_seed(1))
plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
plan.integrate(Fd)
torch.cuda.synchronize()
print("ok")
