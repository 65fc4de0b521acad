"""Where does the GPU barycenter leave the fp64 oracle?  (VERDICT r1 item 1.)

    python tools/bary_trace.py [--iters 10] [--floor 0.0]

Per iteration j of Alg. 1 on the GPU test's inputs
(workloads.barycenter_inputs), three trajectories:
  oracle  fp64 numpy Alg. 1 with FM_K = the fp64 oracle integrator;
  hybrid  the same fp64 iteration with FM_K = the GPU integrate (inputs formed
          exactly as k_sinkhorn.cu forms them);
  gpu     rfd_barycenter run for j iterations.
and, at the oracle's own iterates, the normwise error of one GPU FM_K
application against the oracle's (eta_j, per column max).  Prints
|hybrid - oracle| and |gpu - hybrid| (normwise) per iteration: the first is
the amplification of eta through Alg. 1, the second the elementwise kernels.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import rfd as orf  # noqa: E402
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import barycenter_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--floor", type=float, default=0.0)
a_ = ap.parse_args()

x, a, mus = barycenter_inputs(2000, floor=a_.floor)
eps, lam, m, seed = 0.03, 0.1, 256, 5
plan = rfd.Plan(torch.from_numpy(x).cuda(), eps, lam, m, seed)
ref = orf.Plan(x, eps, lam, m, seed)
a32 = a.astype(np.float32).astype(np.float64)
mus32 = mus.astype(np.float32).astype(np.float64)
alpha = np.array([1 / 3] * 3)


def rel(g, r):
    return float(np.abs(g - r).max() / np.abs(r).max())


def fm_gpu(Z):
    col = (a32[:, None] * Z).max(axis=0)
    s = np.array([2.0 ** -np.frexp(c)[1] if c > 0 else 1.0 for c in col])
    X = ((a32[:, None] * Z) * s[None, :]).astype(np.float32)
    Y = plan.integrate(torch.from_numpy(X).cuda()).cpu().numpy().astype(np.float64)
    return Y / s[None, :]


def fm_ref(Z):
    return ref.apply(a32[:, None] * Z)["out"]


def step(fm, V):
    W = mus32.T / np.maximum(fm(V), 1e-30)
    d = np.maximum(V * fm(W), 1e-30)
    lg = np.zeros(V.shape[0])
    for i in range(V.shape[1]):
        lg = lg + alpha[i] * np.log(d[:, i])
    mu = np.exp(lg)
    return (V * mu[:, None]) / d, mu, W


Vo = np.ones((2000, 3))
Vh = np.ones((2000, 3))
mus_d = torch.from_numpy(mus.astype(np.float32)).cuda()
a_d = torch.from_numpy(a.astype(np.float32)).cuda()
print("iter | eta: GPU FM_K(a v) err, FM_K(a w) err at the oracle's iterate | "
      "hybrid vs oracle | gpu vs hybrid | clamp-bound entries (oracle)")
for j in range(1, a_.iters + 1):
    # one GPU FM_K on the oracle's current inputs
    e1 = rel(fm_gpu(Vo), fm_ref(Vo))
    Wo = mus32.T / np.maximum(fm_ref(Vo), 1e-30)
    e2 = rel(fm_gpu(Wo), fm_ref(Wo))
    clamps = int((fm_ref(Vo) < 1e-30).sum() + (Vo * fm_ref(Wo) < 1e-30).sum())
    Vo, mu_o, _ = step(fm_ref, Vo)
    Vh, mu_h, _ = step(fm_gpu, Vh)
    g, its = plan.barycenter(mus_d, a_d, list(alpha), j)
    g = g.cpu().numpy().astype(np.float64)
    bo, bh = mu_o / (a32 @ mu_o), mu_h / (a32 @ mu_h)
    print("%4d | %.2e %.2e | %.2e | %.2e | %d" % (j, e1, e2, rel(bh, bo), rel(g, bh), clamps))
