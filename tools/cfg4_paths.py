"""cfg-4 integrate time (CUDA-graph replay) by field width: d <= 4 takes the
one-launch narrow kernel, d >= 5 the tensor-core passes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
if len(sys.argv) > 2:  # another build of the library (A/B)
    rfd.load_library(sys.argv[2])
p, x, F = make_config(cfg)
if cfg == 3:
    plan = rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
    x = x.reshape(-1, 3)  # fields: clouds x n rows
else:
    plan = rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
rng = np.random.default_rng(0)
for d in (1, 3, 4, 5, 8, 16):
    Fd = torch.from_numpy(rng.standard_normal((x.shape[0], d)).astype(np.float32)).cuda()
    out = torch.empty_like(Fd)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            plan.integrate(Fd, out=out, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            plan.integrate(Fd, out=out, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 20 * 1e3)
    print("d=%d: %.1f us per integrate (graph, median of 5)" % (d, sorted(ts)[2]), flush=True)
