"""A4 through the spread grid vs the direct tensor-core Gram vs the oracle
(k_nufft.cu).  Usage: python tools/nufft_check.py [n5]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import configs as C  # noqa: E402
from oracle import rfd as orf  # noqa: E402


def relerr(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / np.abs(b).max())


def plan_of(x, p, mode):
    os.environ["RFD_GRAM_SPREAD"] = mode
    torch.cuda.synchronize()
    xd = torch.from_numpy(x).cuda()
    plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    torch.cuda.synchronize()
    return plan


def timed_create(x, p, mode, reps=5):
    os.environ["RFD_GRAM_SPREAD"] = mode
    xd = torch.from_numpy(x).cuda()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
        nodes = plan.info()["gram_nodes"]
        plan.close()
    return min(ts) * 1e3, nodes


def kernel_times(x, p, mode):
    os.environ["RFD_GRAM_SPREAD"] = mode
    xd = torch.from_numpy(x).cuda()
    rfd.profile_enable(True)
    rfd.profile_read()
    for _ in range(3):
        plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
        plan.close()
    torch.cuda.synchronize()
    prof = rfd.profile_read()
    rfd.profile_enable(False)
    return prof


def main():
    rfd.load_library()
    n5 = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    for cfg, n in ((5, n5), (4, None), (2, None)):
        p, x, F = C.make_config(cfg, **({"n": n} if n else {}))
        x = np.ascontiguousarray(x, np.float32)
        ref = orf.Plan(x, p["eps"], p["lam"], p["m"], p["seed"])
        res = ref.apply(F.astype(np.float64))
        for mode in ("0", "2"):
            plan = plan_of(x, p, mode)
            G = plan.export("gram")
            Cc = plan.export("core")
            out = plan.integrate(torch.from_numpy(np.ascontiguousarray(F)).cuda()).cpu().numpy()
            F2 = F.reshape(F.shape[0], -1).astype(np.float64)
            o2 = out.reshape(out.shape[0], -1)
            print(f"cfg{cfg} n={x.shape[0]} mode={mode} nodes={plan.info()["gram_nodes"]} "
                  f"G {relerr(G, ref.G):.2e} C {relerr(Cc, ref.C):.2e} "
                  f"out {relerr(o2, res['out']):.2e} delta {relerr(o2 - F2, res['out'] - F2):.2e}",
                  flush=True)
            plan.close()
    p, x, F = C.make_config(5)
    x = np.ascontiguousarray(x, np.float32)
    for mode in ("0", "1"):
        ms, nodes = timed_create(x, p, mode)
        print(f"cfg5 full plan create mode={mode}: {ms:.3f} ms (wall, min of 5), nodes={nodes}")
        for k, (cnt, tot) in sorted(kernel_times(x, p, mode).items(), key=lambda kv: -kv[1][1]):
            print(f"    {k:24s} {cnt:4d} launches {tot / 3:.4f} ms per plan")
    # determinism
    os.environ["RFD_GRAM_SPREAD"] = "1"
    xd = torch.from_numpy(x).cuda()
    g1 = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"]).export("gram")
    g2 = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"]).export("gram")
    print("bitwise deterministic:", bool(np.array_equal(g1, g2)))


if __name__ == "__main__":
    main()
