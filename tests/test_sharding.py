"""Host logic of the sharded cloud on CPU, world size 2, gloo.

Both sums over points -- G = Phi^T Phi and S = Phi^T F
(Eq. 13) -- are linear in the points, so a cloud split over
ranks needs one all-gather of the partials per sum.  This test runs the
binding's exchange (``rfd.make_allgather``: the very callback the library
calls, here on host buffers over gloo), the row partition
(``rfd.shard_rows``) and the rank-ordered sum k_shard.cu performs, on partials
from the fp64 oracle, and checks:
  * the gathered buffer is rank-major and bitwise the ranks' partials;
  * the rank-ordered sum is bitwise the same on both ranks and equal to the
    single-process sum of the same shard partials in the same order;
  * the merged bounding box / point count equal the whole cloud's;
  * each rank's rows of out = F + Phi C^ S equal the N = 1 oracle's.
The GPU kernels of the same path are covered by the -m gpu tests.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import rfd as orf  # noqa: E402
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather(cb, arr):
    """All-gather a host fp64 array through the library's callback."""
    send = np.ascontiguousarray(arr, np.float64).ravel()
    recv = np.empty(send.size * dist.get_world_size(), np.float64)
    st = cb(None, send.ctypes.data, recv.ctypes.data, send.size, None)
    assert st == 0
    return recv.reshape(dist.get_world_size(), *np.shape(arr))


def _ordered_sum(parts):
    s = parts[0].copy()
    for q in range(1, parts.shape[0]):
        s = s + parts[q]
    return s


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, x, F = make_config(1)
        n = x.shape[0]
        lo, hi = rfd.shard_rows(n, rank, world)
        xl, Fl = x[lo:hi], F[lo:hi].astype(np.float64)
        cb = rfd.make_allgather(None, "cpu")
        omega, _ = orf.frequencies(p["seed"], p["m"])
        nu = orf.importance_weights(omega, p["eps"], orf.l1_ball_mass())
        # bounding box + count exchange (k_shard.cu bbox_export / bbox_merge)
        box = np.concatenate([xl.min(0), xl.max(0), [hi - lo]]).astype(np.float64)
        boxes = _gather(cb, box)
        merged = np.concatenate([boxes[:, :3].min(0), boxes[:, 3:6].max(0)])
        n_total = int(boxes[:, 6].sum())
        # Gram and S partials (the oracle's sums over this rank's points)
        Gl = orf.gram(xl, omega)
        Gparts = _gather(cb, Gl)
        G = _ordered_sum(Gparts)
        C = orf.core(G, nu, p["lam"])
        Sl = orf.project(xl, omega, Fl)
        Sparts = _gather(cb, Sl)
        S = _ordered_sum(Sparts)
        out_l = Fl + orf.features(xl, omega) @ (C @ S)
        q.put(dict(rank=rank, lo=lo, hi=hi, Gl=Gl, Gparts=Gparts, G=G, Sparts=Sparts, S=S,
                   merged=merged, n_total=n_total, out=out_l))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_exchange_and_reduction_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda d: d["rank"])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p, x, F = make_config(1)
    n = x.shape[0]
    omega, _ = orf.frequencies(p["seed"], p["m"])
    # partition: contiguous, covering, sizes within one
    assert [(r["lo"], r["hi"]) for r in res] == [rfd.shard_rows(n, q_, world) for q_ in range(world)]
    assert res[0]["lo"] == 0 and res[-1]["hi"] == n
    assert all(a["hi"] == b["lo"] for a, b in zip(res, res[1:]))
    # gathered buffers are rank-major and bitwise the ranks' own partials
    for r in res:
        for q_ in range(world):
            np.testing.assert_array_equal(r["Gparts"][q_], res[q_]["Gl"])
    # rank-ordered sums: bitwise identical across ranks and to the
    # single-process sum of the same shard partials in rank order
    single_G = _ordered_sum(np.stack([orf.gram(x[r["lo"]:r["hi"]], omega) for r in res]))
    single_S = _ordered_sum(np.stack([orf.project(x[r["lo"]:r["hi"]], omega,
                                                  F[r["lo"]:r["hi"]].astype(np.float64))
                                      for r in res]))
    for r in res:
        np.testing.assert_array_equal(r["G"], single_G)
        np.testing.assert_array_equal(r["S"], single_S)
    # merged bounding box and point count = the whole cloud's
    for r in res:
        np.testing.assert_array_equal(r["merged"], np.concatenate([x.min(0), x.max(0)]).astype(np.float64))
        assert r["n_total"] == n
    # each rank's rows of out match the unsharded oracle
    ref = orf.Plan(x, p["eps"], p["lam"], p["m"], p["seed"]).apply(F)["out"]
    out = np.concatenate([r["out"] for r in res])
    assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()


def test_shard_rows_partition():
    for n, world in ((10, 3), (1024, 8), (7, 7), (5, 2)):
        spans = [rfd.shard_rows(n, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) <= 1 and all(s >= 1 for s in sizes)
