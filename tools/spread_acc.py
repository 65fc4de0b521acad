"""Spread-path G against the oracle on a few clouds, for one build of the
library (A/B of spread-kernel numerics).  python tools/spread_acc.py [lib]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402
from oracle import rfd as orf  # noqa: E402

if len(sys.argv) > 1:
    rfd.load_library(sys.argv[1])
os.environ["RFD_GRAM_SPREAD"] = "2"
rng = np.random.default_rng(5)
cases = []
p, x, _ = make_config(5, n=262144)
cases.append(("cfg5 262k", x, p))
p4, x4, _ = make_config(4)
cases.append(("cfg4", x4, p4))
xp = np.zeros((4096, 3)) + np.array([0.25, -1.0, 3.0])
cases.append(("point", xp.astype(np.float32), dict(eps=0.05, lam=-0.4, m=128, seed=6)))
xm = np.empty((22000, 3))
xm[:9000] = np.array([0.1, 0.2, -0.3])
xm[9000:] = rng.uniform(-0.5, 0.5, (13000, 3))
cases.append(("mass", xm.astype(np.float32), dict(eps=0.05, lam=-0.4, m=128, seed=2)))
for name, x, p in cases:
    ref = orf.Plan(x, p["eps"], p["lam"], p["m"], p["seed"])
    pl = rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
    G = pl.export("gram")
    print("%-10s nodes %6d  G err %.3e" % (name, pl.info()["gram_nodes"],
                                          np.abs(G - ref.G).max() / np.abs(ref.G).max()), flush=True)
