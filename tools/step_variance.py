"""Variance of the timed cfg-5 step loop (20 plan + integrate steps) under the
bench's conditions: per-launch profiling events on/off, the NVML clock-sampler
thread on/off.  python tools/step_variance.py"""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

p, x, F = make_config(5)
xd, Fd = torch.from_numpy(x).cuda(), torch.from_numpy(F).cuda()
out = torch.empty_like(Fd)


def step():
    pl = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    pl.integrate(Fd, out=out)
    pl.close()


class Sampler:
    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(0)
        self.stop = False

    def loop(self):
        while not self.stop:
            self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
            self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            time.sleep(0.05)


for _ in range(3):
    step()
torch.cuda.synchronize()
for prof in (False, True):
    for samp in (False, True):
        res = []
        for rep in range(5):
            s = None
            if samp:
                s = Sampler()
                t = threading.Thread(target=s.loop, daemon=True)
                t.start()
            rfd.profile_enable(prof)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                step()
            e1.record()
            torch.cuda.synchronize()
            rfd.profile_enable(False)
            if s:
                s.stop = True
                t.join()
            res.append(e0.elapsed_time(e1) / 20)
        print("profiling %d sampler %d: ms/step %s" % (prof, samp, " ".join("%.3f" % v for v in res)), flush=True)
