"""Per-call cost of Plan.integrate at cfgs 1, 2, 4: one call between events
(as bench.py's plain loop: host enqueue + device time) and the host time per
call of a 2000-call loop without synchronisation."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

for cfg in (1, 2, 4):
    p, x, F = make_config(cfg)
    xd, Fd = torch.from_numpy(x).cuda(), torch.from_numpy(F).cuda()
    od = torch.empty_like(Fd)
    plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    for _ in range(10):
        plan.integrate(Fd, out=od)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(200):
        e0.record()
        plan.integrate(Fd, out=od)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    t0 = time.perf_counter()
    for _ in range(2000):
        plan.integrate(Fd, out=od)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print("cfg%d one call %.1f us (median), host per call %.1f us" % (cfg, np.median(ts), (t1 - t0) / 2000 * 1e6))
