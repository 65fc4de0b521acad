"""Fused vs unfused rfd_barycenter against the oracle, per iteration count."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import rfd as orf  # noqa: E402
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import barycenter_inputs  # noqa: E402

lam = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
m = int(sys.argv[2]) if len(sys.argv) > 2 else 30
x, a, mus = barycenter_inputs(3000)
plan = rfd.Plan(torch.from_numpy(x).cuda(), 0.03, lam, m, 5)
ref_plan = orf.Plan(x, 0.03, lam, m, 5)
mus_d = torch.from_numpy(mus.astype(np.float32)).cuda()
a_d = torch.from_numpy(a.astype(np.float32)).cuda()


def rel(g, r):
    return float(np.abs(g - r).max() / np.abs(r).max())


for it in (1, 2, 3, 4, 5, 10):
    ref, _ = ref_plan.barycenter(mus, a, [1 / 3] * 3, it)
    os.environ.pop("RFD_BARY_FUSED", None)
    f, _ = plan.barycenter(mus_d, a_d, [1 / 3] * 3, it)
    os.environ["RFD_BARY_FUSED"] = "0"
    u, _ = plan.barycenter(mus_d, a_d, [1 / 3] * 3, it)
    os.environ.pop("RFD_BARY_FUSED", None)
    f = f.cpu().numpy().astype(np.float64)
    u = u.cpu().numpy().astype(np.float64)
    print("it %2d: fused %.2e unfused %.2e fused-vs-unfused %.2e" % (it, rel(f, ref), rel(u, ref), rel(f, u)))
