"""Sharded cloud through the C ABI on ONE GPU (needs a B200).

Two ranks are emulated by two host threads, each with its own plan and
stream; the all-gather callback is a host rendezvous (synchronise the
stream, copy the partial to the host, wait for the other thread, copy the
gathered buffer back).  No kernel waits on another kernel, so this is safe on
one GPU; the NCCL transport itself is torch.distributed's (covered on CPU by
tests/test_sharding.py with gloo).  Checked: every rank holds bitwise the same
G and C^, the merged centre is the whole cloud's, and the concatenated out
rows meet the oracle's N = 1 result at the usual gates.
"""

import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import rfd as orf  # noqa: E402
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402


class _HostGroup:
    def __init__(self, world):
        self.world = world
        self.bufs = [None] * world
        self.bar = threading.Barrier(world)

    def callback(self, rank):
        def cb(_ctx, send, recv, count, stream):
            try:
                st = torch.cuda.ExternalStream(int(stream or 0))
                st.synchronize()
                src = rfd._view(send, count, torch.device("cuda"))
                self.bufs[rank] = src.cpu().clone()
                self.bar.wait(timeout=120)
                gathered = torch.cat(self.bufs).cuda()
                dst = rfd._view(recv, count * self.world, torch.device("cuda"))
                dst.copy_(gathered)
                torch.cuda.synchronize()
                self.bar.wait(timeout=120)
                return 0
            except Exception as e:  # noqa: BLE001
                print("callback failed", e)
                return 1
        return rfd.ALLGATHER_FN(cb)


def _run_ranks(x, F, p, world, d_calls=1):
    grp = _HostGroup(world)
    n = x.shape[0]
    results = [None] * world
    errors = []

    def body(rank):
        try:
            torch.cuda.set_device(0)
            lo, hi = rfd.shard_rows(n, rank, world)
            s = torch.cuda.Stream()
            shard = rfd.Shard(rank, world, grp.callback(rank), None)
            with torch.cuda.stream(s):
                xd = torch.from_numpy(np.ascontiguousarray(x[lo:hi])).cuda()
                Fd = torch.from_numpy(np.ascontiguousarray(F[lo:hi])).cuda()
                plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"], stream=s, _shard=shard)
                for _ in range(d_calls):
                    out = plan.integrate(Fd, stream=s)
                s.synchronize()
            results[rank] = dict(plan=plan, out=out.cpu().numpy(), lo=lo, hi=hi,
                                 G=plan.export("gram"), C=plan.export("core"), info=plan.info())
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            grp.bar.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errors, errors
    return results


def _relerr(got, ref):
    return float(np.abs(np.asarray(got, np.float64) - ref).max() / np.abs(ref).max())


@pytest.mark.parametrize("cfg,world,spread", [(2, 2, "1"), (4, 3, "1"), (1, 2, "1"), (4, 2, "2")])
def test_sharded_cloud_matches_oracle(cfg, world, spread, monkeypatch):
    # spread "2": every rank's partial G through the spread grid (k_nufft.cu)
    # on the merged bounding box
    monkeypatch.setenv("RFD_GRAM_SPREAD", spread)
    p, x, F = make_config(cfg)
    res = _run_ranks(x, F, p, world, d_calls=2)
    ref = orf.Plan(x, p["eps"], p["lam"], p["m"], p["seed"])
    for r in res:
        assert r["info"]["n_total"] == x.shape[0] and r["info"]["world"] == world
        assert (r["info"]["gram_nodes"] > 0) == (spread == "2")
        np.testing.assert_array_equal(r["G"], res[0]["G"])  # same bits on every rank
        np.testing.assert_array_equal(r["C"], res[0]["C"])
    eG, eC = _relerr(res[0]["G"], ref.G), _relerr(res[0]["C"], ref.C)
    out = np.concatenate([r["out"] for r in res])
    oref = ref.apply(F.astype(np.float64))["out"]
    eo = _relerr(out, oref)
    ed = _relerr(out - F, oref - F)
    print("sharded cfg%d world %d: G %.2e C %.2e out %.2e delta %.2e" % (cfg, world, eG, eC, eo, ed))
    assert max(eG, eC, eo, ed) <= 1e-4


def test_sharded_single_rank_equals_plain_plan():
    # world = 1 (no exchange): bitwise the plain plan
    p, x, F = make_config(2)
    xd, Fd = torch.from_numpy(x).cuda(), torch.from_numpy(F).cuda()
    a = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"]).integrate(Fd)
    b = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"],
                 _shard=rfd.Shard(0, 1, rfd.ALLGATHER_FN(), None)).integrate(Fd)
    assert torch.equal(a, b)
