"""Phase timestamps of the d <= 4 one-launch integrate (RFD_SMALL_TRACE=1) per config."""
import os
import sys

os.environ["RFD_SMALL_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

for cfg in (1, 2, 4, 3):
    p, x, F = make_config(cfg)
    if cfg == 3:
        F = F[0]
    plan = rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
    Fd = torch.from_numpy(F).cuda()
    for _ in range(3):
        plan.integrate(Fd)
    torch.cuda.synchronize()
    print("cfg", cfg, flush=True)
