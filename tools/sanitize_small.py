"""Small runs of the main paths for compute-sanitizer (memcheck / racecheck):
cfg 1 (narrow kernel), and 16k cfg-5-recipe points with m = 128, d = 16
through rfd_gfi with the spread-grid Gram forced (spread, grid Gram, core,
tensor-core passes)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

p, x, F = make_config(1)
plan = rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
o1 = plan.integrate(torch.from_numpy(F).cuda())
os.environ["RFD_GRAM_SPREAD"] = "2"
p, x, F = make_config(5, n=16384)
out = rfd.gfi(torch.from_numpy(x).cuda(), p["eps"], p["lam"], 128, p["seed"], torch.from_numpy(F).cuda())
torch.cuda.synchronize()
print("ok", float(o1.abs().max()), float(out.abs().max()))
