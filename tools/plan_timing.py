"""Wall-clock distribution of cfg-5 plan creation (host view, includes the
library's host synchronisations), and of plan + integrate steps.

    python tools/plan_timing.py [reps]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
p, x, F = make_config(5)
xd, Fd = torch.from_numpy(x).cuda(), torch.from_numpy(F).cuda()
out = torch.empty_like(Fd)
for _ in range(3):
    rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"]).close()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    t = time.perf_counter()
    pl = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    ts.append(time.perf_counter() - t)
    pl.close()
ts = np.array(ts) * 1e3
print("plan create ms: min %.3f p10 %.3f p50 %.3f p90 %.3f max %.3f" % tuple(np.percentile(ts, [0, 10, 50, 90, 100])))
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st = []
for _ in range(reps):
    torch.cuda.synchronize()
    ev0.record()
    pl = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    pl.integrate(Fd, out=out)
    ev1.record()
    torch.cuda.synchronize()
    st.append(ev0.elapsed_time(ev1))
    pl.close()
st = np.array(st)
print("step ms (events): min %.3f p10 %.3f p50 %.3f p90 %.3f max %.3f" % tuple(np.percentile(st, [0, 10, 50, 90, 100])))
