"""The degenerate 'point' cloud through the spread-grid Gram (debug helper)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_00942_b200 import rfd  # noqa: E402

os.environ["RFD_GRAM_SPREAD"] = "2"
os.environ.setdefault("RFD_SYNC_CHECK", "1")
n = 4096
x = (np.zeros((n, 3)) + np.array([0.25, -1.0, 3.0])).astype(np.float32)
F = np.random.default_rng(11).standard_normal((n, 8)).astype(np.float32)
plan = rfd.Plan(torch.from_numpy(x).cuda(), 0.05, -0.4, 128, 6)
print("nodes", plan.info()["gram_nodes"], flush=True)
out = plan.integrate(torch.from_numpy(F).cuda())
torch.cuda.synchronize()
print("ok", float(out.abs().max()))
