"""Pinned-host copy bandwidth on the box: H2D alone, D2H alone, both at once
(two streams), and rfd_gfi_host at cfg 5 with 1 / 2 / 3 calls in flight."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

nb = 318 * 2**20
h = torch.empty(nb // 4, dtype=torch.float32).pin_memory()
h2 = torch.empty(nb // 4, dtype=torch.float32).pin_memory()
d = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
d2 = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def bw(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = bw(fn)
    print("%-5s %.3f ms  %.1f GB/s per direction" % (name, ms, nb / ms / 1e6))

p, x, F = make_config(5)
for nslot in (1, 2, 3):
    xh = [torch.from_numpy(x).pin_memory() for _ in range(nslot)]
    Fh = [torch.from_numpy(F).pin_memory() for _ in range(nslot)]
    oh = [torch.empty_like(Fh[0]).pin_memory() for _ in range(nslot)]
    streams = [torch.cuda.Stream() for _ in range(nslot)]

    def call(i):
        k = i % nslot
        rfd.gfi_host(xh[k], p["eps"], p["lam"], p["m"], p["seed"], Fh[k], oh[k], stream=streams[k])

    for i in range(4):
        call(i)
    torch.cuda.synchronize()
    main = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for s in streams:
        s.wait_event(e0)
    K = 12
    for i in range(K):
        call(i)
    for s in streams:
        main.wait_stream(s)
    e1.record(main)
    torch.cuda.synchronize()
    print("gfi_host %d in flight: %.3f ms/step" % (nslot, e0.elapsed_time(e1) / K))
