"""Per-call device time of rfd_integrate at cfgs 1-4 from CUDA-graph replays."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

if len(sys.argv) > 1:  # another build of the library (A/B)
    rfd.load_library(sys.argv[1])

for cfg in (1, 2, 4, 3):
    p, x, F = make_config(cfg)
    if cfg == 3:
        F = F[0]
    plan = rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
    Fd = torch.from_numpy(np.ascontiguousarray(F)).cuda()
    od = torch.empty_like(Fd)
    s2 = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s2):
        plan.integrate(Fd, out=od, stream=s2)
        with torch.cuda.graph(g, stream=s2):
            for _ in range(50):
                plan.integrate(Fd, out=od, stream=s2)
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 50 * 1e3)
    print("cfg%d graph %.1f us per integrate (coop=%s)" % (cfg, float(np.median(ts)), os.environ.get("RFD_SMALL_COOP", "1")))
