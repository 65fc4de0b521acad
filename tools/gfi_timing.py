"""cfg-5 step: rfd_plan_create + rfd_integrate vs the one-shot rfd_gfi (pass 1
beside the core), CUDA events over 20 steps, 5 repetitions each."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

if len(sys.argv) > 1:  # another build of the library (A/B)
    rfd.load_library(sys.argv[1])
p, x, F = make_config(5)
xd, Fd = torch.from_numpy(x).cuda(), torch.from_numpy(F).cuda()
out = torch.empty_like(Fd)


def two_calls():
    pl = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    pl.integrate(Fd, out=out)
    pl.close()


def one_shot():
    rfd.gfi(xd, p["eps"], p["lam"], p["m"], p["seed"], Fd, out=out)


for name, fn in (("plan+integrate", two_calls), ("gfi", one_shot)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    res = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 20)
    print("%-15s ms/step %s" % (name, " ".join("%.3f" % v for v in res)), flush=True)
