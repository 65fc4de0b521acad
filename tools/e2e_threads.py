"""e2e (rfd_gfi_host, pinned host buffers) with 2 calls in flight: one host
thread issuing both slots vs one host thread per slot."""
import os
import sys
import threading

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

p, x, F = make_config(5)
K = 20
nslot = 2
xh = [torch.from_numpy(x).pin_memory() for _ in range(nslot)]
Fh = [torch.from_numpy(F).pin_memory() for _ in range(nslot)]
oh = [torch.empty_like(Fh[0]).pin_memory() for _ in range(nslot)]
main = torch.cuda.current_stream()
streams = [torch.cuda.Stream() for _ in range(nslot)]


def call(k):
    rfd.gfi_host(xh[k], p["eps"], p["lam"], p["m"], p["seed"], Fh[k], oh[k], stream=streams[k])


def timed(threaded):
    for i in range(4):
        call(i % nslot)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for s in streams:
        s.wait_event(e0)
    if threaded:
        def run(k):
            torch.cuda.set_device(0)
            for _ in range(K // nslot):
                call(k)
        ts = [threading.Thread(target=run, args=(k,)) for k in range(nslot)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    else:
        for i in range(K):
            call(i % nslot)
    for s in streams:
        main.wait_stream(s)
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


for rep in range(3):
    print("single thread %.3f ms/step   thread per slot %.3f ms/step" % (timed(False), timed(True)),
          flush=True)
