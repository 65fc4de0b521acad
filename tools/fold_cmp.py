import os, sys
import numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from paper_2302_00942_b200 import rfd
import oracle.rfd as orf
for nc, nu in ((20000, 2000), (9000, 13000), (12000, 20000)):
  rng = np.random.default_rng(5)
  n = nc + nu
  x = np.empty((n, 3)); x[:nc] = np.array([0.1, 0.2, -0.3]); x[nc:] = rng.uniform(-0.5, 0.5, (nu, 3)); x = x.astype(np.float32)
  F = rng.standard_normal((n, 4)).astype(np.float32)
  p = dict(eps=0.05, lam=-0.4, m=128, seed=2)
  print("coincident", nc, "uniform", nu)
  ref = orf.Plan(x, p["eps"], p["lam"], p["m"], p["seed"])
  res = ref.apply(F.astype(np.float64))
  def rel(a, b): return np.abs(a - b).max() / np.abs(b).max()
  for mode in ("0", "2"):
      os.environ["RFD_GRAM_SPREAD"] = mode
      pl = rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
      out = pl.integrate(torch.from_numpy(F).cuda()).cpu().numpy()
      print(mode, pl.info()["gram_nodes"], "G %.2e C %.2e out %.2e delta %.2e" % (rel(pl.export("gram"), ref.G), rel(pl.export("core"), ref.C), rel(out, res["out"]), rel(out - F, res["out"] - F)))
