"""Benchmark of the RFD hot path on B200 (contract: see DESIGN.md Sec. 8).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl rfd|reference]

One STEP = one pass of the whole hot path over
the BASELINE.json scoring config (cfg 5: N = 4,194,304 points in the unit
cube, m = 256, d = 16, eps = 0.01, lambda = -0.3): rfd_plan_create
(frequencies, Gram, core) + rfd_integrate (pass 1, Y, pass 2), inputs
resident in HBM.  value = N * d * steps * ranks / max-over-ranks time
(points x dims / s).  Multi-GPU: ONE
cloud of ranks x 4M points sharded over the ranks (rfd_plan_create_sharded);
the Gram and S partials are all-gathered over NCCL (torch.distributed) and
summed in rank order by the library -- weak scaling (4M points per GPU).
``--gpus N`` without torchrun re-launches itself under torch.distributed.run.

Extra keys: ``integrate`` (inference only, plan reused: the paper's
"inference"), ``roofline`` for the dominant kernel (timed with
CUDA events on its launch stream inside the timed region), ``kernels`` (every
kernel's share), ``e2e`` (host buffers through the C ABI), ``cpu_baseline``
(the fp64 oracle on a bounded sample, rank 0, N = 1 only), ``clocks`` (NVML
samples during the timed region), ``gpu_launches``.
"""

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import make_config  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
# B200 unit counts (B200_PROFILING.md: 148 SMs, clocks.max.sm 1965 MHz; CUDA
# throughput table for cc 10.0: 128 FP32 FMA and 16 MUFU results / clk / SM).
SMS, FMA_PER_CLK, MUFU_PER_CLK = 148, 128, 16
SPREAD_WIDTH = 8   # a4 spread-grid kernel width (csrc/rfd_internal.h kNufftWidth)
METRIC = "GFI points x dims / s (RFD plan + integrate, cfg5 N=4M m=256 d=16)"
UNIT = "points*dims/s"


def peaks():
    p = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "bf16_tflops": 1590.0,
         "src": "fallback (B200_PROFILING.md)"}
    if os.path.exists(PEAKS_PATH):
        with open(PEAKS_PATH) as f:
            j = json.load(f)
        p.update({k: j[k] for k in ("hbm_gbs", "sm_max_mhz", "bf16_tflops") if k in j})
        p["src"] = "measured (MEASURED_PEAKS.json)"
    return p


# ------------------------------------------------------------------ work model
# Peaks: FP32 FMA pipe and MUFU from the B200 unit counts at
# sm_max_mhz; dense fp16 tensor = the measured bf16 burst (same rate for fp16),
# tf32 = half of it (the guide's nominal 1.1 vs 2.25 PFLOP/s ratio).
def kernel_work(name, N, m, d, nodes=0):
    """Algorithmic work of one launch: dict of {fma, mufu, bytes, tensor_flop, tensor_kind}.

    Algorithmic = what the method needs, not what the kernel
    executes: the 3-product hi/lo splits, masked tile halves, range reduction
    and loop control count against achieved efficiency, not the roofline.
    nodes > 0: a4 went through the spread grid (k_nufft.cu):
    the tensor-core Gram runs over the grid's nodes, the spread kernel does
    W^3 multiply-adds and 3W kernel values (rsqrt + ex2, ~6 FMA) per point,
    W = SPREAD_WIDTH.
    """
    r = 2 * m
    dc = min(d, 16)
    if name in ("rfd_gram_partial", "rfd_gram_tc"):   # G = Phi^T Phi (upper triangle)
        Ng = nodes if nodes > 0 else N
        w = dict(fma=Ng * r * (r + 1) / 2 + 3.0 * Ng * m, mufu=2.0 * Ng * m, bytes=16.0 * Ng,
                 proj=3.0 * Ng * m)
        if name == "rfd_gram_tc":
            w.update(tensor_flop=2.0 * Ng * r * (r + 1) / 2, tensor_kind="f16")
        return w
    if name == "rfd_nufft_spread" and nodes > 0:
        W = SPREAD_WIDTH
        return dict(fma=N * (W ** 3 + 3.0 * W * 6), mufu=2.0 * 3 * W * N,
                    bytes=20.0 * N + 8.0 * nodes)
    if name in ("rfd_pass1", "rfd_pass1_tc"):           # S = Phi^T F
        w = dict(fma=2.0 * N * m * dc + 3.0 * N * m, mufu=2.0 * N * m, bytes=N * (16 + 4 * dc),
                 proj=3.0 * N * m)
    elif name in ("rfd_pass2", "rfd_pass2_tc"):         # out = F + Phi Y
        w = dict(fma=2.0 * N * m * dc + 3.0 * N * m, mufu=2.0 * N * m, bytes=N * (16 + 8 * dc),
                 proj=3.0 * N * m)
    else:
        return None
    if name.endswith("_tc"):
        w.update(tensor_flop=2.0 * 2.0 * N * m * dc, tensor_kind="tf32")
    return w


def peaks_of(pk):
    clk = pk["sm_max_mhz"] * 1e6
    bf16 = pk.get("bf16_tflops", 1590.0) * 1e12
    return {"fma": SMS * FMA_PER_CLK * clk, "mufu": SMS * MUFU_PER_CLK * clk,
            "hbm": pk["hbm_gbs"] * 1e9, "f16": bf16, "tf32": bf16 / 2}


def ncu_traffic(name):
    """DRAM bytes per launch of kernel `name` from the committed `ncu --set full`
    capture of this workload (profiles/traffic.json, written by
    tools/save_profiles.sh via tools/ncu_traffic.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            e = json.load(f).get(name)
        return None if e is None else float(e["bytes_per_launch"])
    except (OSError, ValueError, KeyError):
        return None


def roofline_of(name, N, m, d, ms_per_launch, pk, nodes=0):
    """Roofline of one kernel: the slowest of its algorithmic HBM bytes, tensor
    flops (tensor-core kernels: the contraction runs there) or FP32 FMA (SIMT
    kernels), and MUFU work, each at its peak.  MUFU-bound kernels report
    bound "alu" (pipe "mufu") against the derived 148 x 16/clk peak."""
    w = kernel_work(name, N, m, d, nodes)
    if w is None or ms_per_launch <= 0:
        return None
    P = peaks_of(pk)
    t = ms_per_launch * 1e-3
    terms = {"hbm": w["bytes"] / P["hbm"], "sfu": w["mufu"] / P["mufu"]}
    if "tensor_flop" in w:
        terms["tensor"] = w["tensor_flop"] / P[w["tensor_kind"]]
        terms["alu"] = w["proj"] / P["fma"]            # projections only
    else:
        terms["alu"] = w["fma"] / P["fma"]
    bound = max(terms, key=terms.get)
    t_roof = terms[bound]
    out = {"bound": bound, "frac": t_roof / t, "traffic": ncu_traffic(name),
           "traffic_note": "DRAM read+write bytes per launch, ncu --set full of tools/profile_step.py "
                           "(cfg 5; profiles/traffic.json); algorithmic bytes per launch: %.4g" % w["bytes"],
           "terms_ms": {k: v * 1e3 for k, v in terms.items()}}
    if bound == "hbm":
        out.update(achieved=w["bytes"] / t / 1e9, peak=P["hbm"] / 1e9, unit="GB/s")
    elif bound == "tensor":
        out.update(achieved=w["tensor_flop"] / t / 1e12, peak=P[w["tensor_kind"]] / 1e12,
                   unit="TFLOP/s", peak_note="dense %s tensor: measured bf16 burst%s"
                   % (w["tensor_kind"], " / 2 (tf32 nominal ratio)" if w["tensor_kind"] == "tf32" else ""))
    elif bound == "alu":
        out.update(achieved=2 * w["fma"] / t / 1e12, peak=2 * P["fma"] / 1e12, unit="TFLOP/s",
                   peak_note="fp32 FMA pipe: 148 SM x 128 FMA/clk x %.0f MHz (derived)" % pk["sm_max_mhz"])
    else:
        out.update(bound="alu", pipe="mufu", achieved=w["mufu"] / t / 1e12, peak=P["mufu"] / 1e12,
                   unit="Tops/s",
                   peak_note="MUFU sin/cos: 148 SM x 16/clk x %.0f MHz (derived, DESIGN.md Sec. 6)"
                   % pk["sm_max_mhz"])
    return out


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML samples of SM clock and throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, device_index):
        self.ok = False
        self.samples = []
        self.reasons = set()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = self._handle(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # no NVML: report it, keep timing on the device
            self.err = str(e)

    def _handle(self, idx):
        # NVML indexes physical GPUs; map through CUDA_VISIBLE_DEVICES.
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        toks = [t.strip() for t in vis.split(",") if t.strip()]
        if toks and idx < len(toks) and toks[idx].isdigit():
            return self.nv.nvmlDeviceGetHandleByIndex(int(toks[idx]))
        if toks and idx < len(toks) and toks[idx].startswith("GPU-"):
            return self.nv.nvmlDeviceGetHandleByUUID(toks[idx])
        return self.nv.nvmlDeviceGetHandleByIndex(idx)

    def _loop(self):
        while not self.stop:
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        self.stop = False
        if self.ok:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self.stop = True
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": self.err}
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------ arms
def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != world:
        if world == 1 and "RANK" not in os.environ:  # spawn the N ranks ourselves
            import socket
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                port = so.getsockname()[1]
            os.execvp(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                       "--nproc-per-node=%d" % args.gpus, "--master-addr",
                                       "127.0.0.1", "--master-port", str(port),
                                       os.path.abspath(__file__)] + sys.argv[1:])
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "rfd" else "gloo"
        if args.impl == "rfd":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
        pg = dist
    elif args.impl == "rfd":
        torch.cuda.set_device(0)
    return rank, world, local, pg


def max_over_ranks(val, pg):
    if pg is None:
        return val
    import torch
    t = torch.tensor([val], dtype=torch.float64, device="cuda" if pg.get_backend() == "nccl" else "cpu")
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def barrier(pg):
    if pg is not None:
        pg.barrier()


def run_rfd(args, rank, world, local, pg):
    import torch
    from paper_2302_00942_b200 import rfd

    p, x, F = make_config(5)
    if rank > 0:  # rank r's shard of the one cloud: 4M more uniform cube points
        rng = np.random.default_rng(4 + 1000 * rank)
        x = rng.random(x.shape, dtype=np.float32)
        F = rng.standard_normal(F.shape, dtype=np.float32)
    N, m, d = p["n"], p["m"], p["d"]
    seed = p["seed"]
    stream = torch.cuda.current_stream()

    def make_plan(points):
        if world > 1:
            return rfd.Plan.sharded(points, p["eps"], p["lam"], m, seed)
        return rfd.Plan(points, p["eps"], p["lam"], m, seed)
    xd = torch.from_numpy(x).cuda()
    Fd = torch.from_numpy(F).cuda()
    outd = torch.empty_like(Fd)
    pk = peaks()

    def step_seq():  # the two calls one after the other
        plan = make_plan(xd)
        plan.integrate(Fd, out=outd)
        plan.close()

    def step():
        if world > 1:
            step_seq()
        else:  # one-shot GFI: pass 1 beside the plan's core (bitwise the two calls)
            rfd.gfi(xd, p["eps"], p["lam"], m, seed, Fd, out=outd)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- per-kernel breakdown (untimed): K steps with every launch bracketed
    # by events; it names the dominant kernel, which alone is bracketed in the
    # timed region (events around every launch add ~8 % to the step: they sit
    # between programmatically dependent launches).  The breakdown runs the
    # same kernels one after the other (rfd_plan_create + rfd_integrate), so
    # the shares add up; the timed step overlaps pass 1 with the core (rfd_gfi).
    rfd.profile_only(None)
    rfd.profile_enable(True)
    rfd.profile_read()
    for _ in range(args.steps):
        step_seq()
    prof_all = rfd.profile_read()
    rfd.profile_enable(False)
    dom = max(prof_all.items(), key=lambda kv: kv[1][1])[0]

    # ---- timed region: K full steps
    sampler = ClockSampler(torch.cuda.current_device())
    rfd.profile_only(dom)
    rfd.profile_enable(True)
    rfd.profile_read()
    l0 = rfd.launch_count()
    barrier(pg)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)] \
            if args.step_times else None
        ev0.record(stream)
        for i in range(args.steps):
            if evs:
                evs[i].record(stream)
            step()
        if evs:
            evs[-1].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        if evs:
            print("step ms:", " ".join("%.3f" % evs[i].elapsed_time(evs[i + 1])
                                       for i in range(args.steps)), file=sys.stderr)
    barrier(pg)
    launches = rfd.launch_count() - l0
    prof_dom = rfd.profile_read()
    rfd.profile_enable(False)
    rfd.profile_only(None)
    ms = ev0.elapsed_time(ev1)
    ms_max = max_over_ranks(ms, pg)
    ms_step = ms_max / args.steps

    # ---- inference only (plan reused), same protocol
    plan = make_plan(xd)
    gram_nodes = int(plan.info()["gram_nodes"])  # a4 via the spread grid (0: direct)
    for _ in range(args.warmup):
        plan.integrate(Fd, out=outd)
    torch.cuda.synchronize()
    barrier(pg)
    # (an extra key, not the contract's value: K steps timed three times, the
    # median reported -- single runs varied by ~4 % between otherwise equal runs)
    ims_runs = []
    for _ in range(3):
        ev0.record(stream)
        for _ in range(args.steps):
            plan.integrate(Fd, out=outd)
        ev1.record(stream)
        torch.cuda.synchronize()
        ims_runs.append(max_over_ranks(ev0.elapsed_time(ev1), pg) / args.steps)
    ims = sorted(ims_runs)[1]
    rfd.profile_enable(True)
    rfd.profile_read()
    for _ in range(args.steps):
        plan.integrate(Fd, out=outd)
    iprof = rfd.profile_read()
    rfd.profile_enable(False)

    # ---- re-parameterisation: nu + core on the stored G.
    # The call reads back the scaling exponent and an overflow flag, so its
    # time includes two device->host round trips.
    rts = []
    for i in range(0 if args.no_configs else args.warmup + args.steps):
        torch.cuda.synchronize()
        ev0.record(stream)
        plan.reparam(p["eps"] * (1.0 + 0.25 * (i % 2)), p["lam"])
        ev1.record(stream)
        torch.cuda.synchronize()
        if i >= args.warmup:
            rts.append(ev0.elapsed_time(ev1))
    # ---- spectrum: k = 32 smallest eigenvalues of exp(lambda W~)
    sts = []
    for i in range(0 if args.no_configs else 2 + 3):
        torch.cuda.synchronize()
        ev0.record(stream)
        plan.spectrum(32)
        ev1.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            sts.append(ev0.elapsed_time(ev1))
    spectrum = None if not sts else {"ms_per_call": float(np.median(sts)), "k": 32,
                "note": "rfd_plan_spectrum at cfg5 (r = 512): Householder tridiagonalisation "
                        "of D^1/2 G D^1/2 in fp64 + bisection, median of 3"}
    reparam = None if not rts else {"ms_per_call": float(np.median(rts)),
               "plan_create_ms": ms_step - ims,
               "note": "rfd_plan_reparam(eps, lambda) at cfg5: nu + core on the stored Gram "
                       "(median of %d); plan_create_ms = step - integrate" % len(rts)}
    plan.close()

    # ---- end to end through the public API with host buffers
    # Every step: points + F copied from pinned host memory, out copied back.
    # Single GPU: rfd_gfi_host (F's upload overlaps the plan, out's download
    # overlaps pass 2), two calls in flight on two streams with their own
    # buffers -- as a serving loop runs it -- so one step's download overlaps
    # the next step's upload (PCIe is full duplex); "serial_ms_per_step" is one
    # stream, one call at a time.
    e2e = None
    if not args.no_e2e:
        nslot = 2 if world == 1 else 1
        xh = [torch.from_numpy(x).pin_memory() for _ in range(nslot)]
        Fh = [torch.from_numpy(F).pin_memory() for _ in range(nslot)]
        oh = [torch.empty_like(Fh[0]).pin_memory() for _ in range(nslot)]
        streams = [stream] + [torch.cuda.Stream() for _ in range(nslot - 1)]

        def e2e_step(i):
            k = i % nslot
            if world > 1:
                pl = make_plan(xh[k])                         # H2D of the points inside
                pl.integrate_host(Fh[k], oh[k])              # H2D F, integrate, D2H out
                pl.close()
            else:
                rfd.gfi_host(xh[k], p["eps"], p["lam"], m, seed, Fh[k], oh[k], stream=streams[k])

        def timed_e2e(slots):
            for i in range(max(1, args.warmup)):
                e2e_step(i if slots > 1 else 0)
            torch.cuda.synchronize()
            barrier(pg)
            ev0.record(stream)
            for s_ in streams[1:slots]:
                s_.wait_event(ev0)
            for i in range(args.steps):
                e2e_step(i if slots > 1 else 0)
            for s_ in streams[1:slots]:
                stream.wait_stream(s_)
            ev1.record(stream)
            torch.cuda.synchronize()
            return max_over_ranks(ev0.elapsed_time(ev1), pg) / args.steps

        ems_serial = timed_e2e(1)
        ems = timed_e2e(nslot)
        e2e = {"value": N * d * world / (ems * 1e-3), "unit": UNIT,
               "ms_per_step": ems, "serial_ms_per_step": ems_serial,
               "h2d_bytes_per_step": int(xh[0].numel() * 4 + Fh[0].numel() * 4),
               "d2h_bytes_per_step": int(oh[0].numel() * 4),
               "api": ("rfd_gfi_host (points + F from pinned host memory, out to pinned host memory), "
                       "%d calls in flight on %d streams" % (nslot, nslot))
                      if world == 1 else "rfd_plan_create_sharded + rfd_integrate_host"}

    # ---- kernels (untimed breakdown pass), dominant kernel roofline (timed region)
    prof = prof_all
    total = sum(v[1] for v in prof.values()) or 1.0
    kernels = {}
    for name, (cnt, tms) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        per = tms / cnt
        kernels[name] = {"launches": cnt, "ms_per_launch": per, "share": tms / total}
        rl = roofline_of(name, N, m, d, per, pk, gram_nodes)
        if rl:
            kernels[name]["roofline_frac"] = rl["frac"]
            kernels[name]["bound"] = rl.get("pipe", rl["bound"])
    dcnt, dms = prof_dom.get(dom, prof[dom])
    roof = roofline_of(dom, N, m, d, dms / dcnt, pk, gram_nodes) or {}
    roof = dict(roof, kernel=dom, peak_src=pk["src"], launches_timed=dcnt,
                timing="CUDA events around each launch of this kernel inside the timed region "
                       "(the other kernels' breakdown: an untimed pass of the same K steps with "
                       "the kernels one after the other)")
    if dom == "rfd_gram_tc" and gram_nodes == 0 and 2 * m >= 256 and roof.get("unit") == "TFLOP/s":
        # What the kernel executes: per 256 x 256 pair tile and point, 2 (diagonal)
        # or 3 (off-diagonal) fp16 products of the hi/lo split (Gram):
        # even at a fully busy tensor pipe frac cannot exceed algorithmic/executed.
        T2 = (2 * m + 255) // 256
        ex = 2.0 * 256 * 256 * N * (2 * T2 + 3 * T2 * (T2 - 1) // 2)
        alg = kernel_work(dom, N, m, d)["tensor_flop"]
        t = dms / dcnt * 1e-3
        roof.update(executed_tflop_per_s=ex / t / 1e12, split_ceiling_frac=alg / ex,
                    executed_frac=ex / t / 1e12 / roof["peak"])

    ikern = {}
    itotal = sum(v[1] for v in iprof.values()) or 1.0
    for name, (cnt, tms) in iprof.items():
        rl = roofline_of(name, N, m, d, tms / cnt, pk)
        ikern[name] = {"ms_per_launch": tms / cnt, "share": tms / itotal,
                       "roofline_frac": rl["frac"] if rl else None}
    # integrate roofline (north star: slower of HBM bytes and FMA+SFU work;
    # SURVEY Sec. 8(d)).  Headline: the contraction counted as FP32 FMA.  Because
    # the contraction runs on the tensor cores, the stricter max(HBM, tensor,
    # MUFU) roofline is reported beside it.
    P = peaks_of(pk)
    fma_i = N * (4.0 * m * d + 6.0 * m)
    mufu_i = 4.0 * N * m
    byts_i = N * (24.0 + 12.0 * d)
    tc_i = 2.0 * 4.0 * N * m * d
    t_roof = max(fma_i / P["fma"], mufu_i / P["mufu"], byts_i / P["hbm"])
    t_strict = max(tc_i / P["tf32"], mufu_i / P["mufu"], byts_i / P["hbm"])
    integ = {"value": N * d * world / (ims * 1e-3), "unit": UNIT, "ms_per_call": ims,
             "ms_per_call_runs": ims_runs,
             "roofline_ms": t_roof * 1e3, "roofline_frac": t_roof / (ims * 1e-3),
             "roofline_bound": "fp32 FMA pipe (4md+6m FMA/pt at 148x128/clk, %.0f MHz)" % pk["sm_max_mhz"],
             "strict_roofline_ms": t_strict * 1e3, "strict_roofline_frac": t_strict / (ims * 1e-3),
             "strict_roofline_bound": "MUFU (4m sin/cos per pt at 148x16/clk) vs tf32 tensor vs HBM",
             "hbm_gbs_achieved": byts_i / (ims * 1e-3) / 1e9, "kernels": ikern}
    return dict(N=N, m=m, d=d, ms_step=ms_step, launches=launches, roofline=roof,
                kernels=kernels, integrate=integ, e2e=e2e, clocks=sampler.summary(), params=p,
                reparam=reparam, spectrum=spectrum, gram_nodes=gram_nodes)


def config_legs(args, pk):
    """SURVEY 8(d) per-config timing: integrate at cfgs 1, 2, 4 (median of
    timed calls) against each config's roofline, the cfg-3 reuse loop (50
    applications over 256 clouds, plain and CUDA-graph captured), and the
    eps-independence check at cfg 5."""
    import torch
    from paper_2302_00942_b200 import rfd
    P = peaks_of(pk)
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def roof(N, m, d):
        t = max(2.0 * 4.0 * N * m * d / P["tf32"], 4.0 * N * m / P["mufu"],
                N * (24.0 + 12.0 * d) / P["hbm"])
        return t * 1e3

    def timed(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            ev0.record(stream)
            fn()
            ev1.record(stream)
            torch.cuda.synchronize()
            ts.append(ev0.elapsed_time(ev1))
        return float(np.median(ts)), float(np.percentile(ts, 10)), float(np.percentile(ts, 90))

    out = {}
    for cfg in (1, 2, 4):
        p, x, F = make_config(cfg)
        xd, Fd = torch.from_numpy(x).cuda(), torch.from_numpy(F).cuda()
        od = torch.empty_like(Fd)
        mk = lambda: rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"]).close()  # noqa: E731
        pmed = timed(mk, 5)[0]
        plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
        med, p10, p90 = timed(lambda: plan.integrate(Fd, out=od), 200)
        # the same calls captured in a CUDA graph (20 per replay): device time
        # without the per-call host cost (ctypes + launch) that bounds the
        # plain loop for these sizes
        s2 = torch.cuda.Stream()
        s2.wait_stream(stream)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s2):
            plan.integrate(Fd, out=od, stream=s2)
            with torch.cuda.graph(gr, stream=s2):
                for _ in range(20):
                    plan.integrate(Fd, out=od, stream=s2)
        torch.cuda.synchronize()
        gmed = timed(gr.replay, 20)[0] / 20
        N, m, d = p["n"], p["m"], p["d"]
        rl = roof(N, m, d)
        out["cfg%d" % cfg] = {"integrate_us": med * 1e3, "p10_us": p10 * 1e3, "p90_us": p90 * 1e3,
                              "graph_us": gmed * 1e3,
                              "value": N * d / (gmed * 1e-3), "unit": UNIT,
                              "strict_roofline_us": rl * 1e3, "strict_roofline_frac": rl / gmed,
                              "plan_create_ms": pmed,
                              "path": ("rfd_integrate_small (one cooperative launch)"
                                       if (d == 1 or N <= 4096 or N > 65536) else
                                       "tensor-core passes (pass 1, a7 fused into pass 2)")}
        plan.close()
        del gr
    # cfg 3: 50 applications back to back on device-resident vectors
    p, x, V = make_config(3)
    xd = torch.from_numpy(x).cuda()
    pmed3 = timed(lambda: rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"]).close(), 5)[0]
    plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    Vd = torch.from_numpy(V).cuda()
    outs = torch.empty_like(Vd)
    A = p["applications"]

    def loop():
        for t in range(A):
            plan.integrate(Vd[t], out=outs[t])
    med, p10, p90 = timed(loop, 10)
    s2 = torch.cuda.Stream()
    s2.wait_stream(stream)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s2):
        plan.integrate(Vd[0], out=outs[0])
        with torch.cuda.graph(g, stream=s2):
            for t in range(A):
                plan.integrate(Vd[t], out=outs[t], stream=s2)
    torch.cuda.synchronize()
    gmed, gp10, gp90 = timed(g.replay, 10)
    Ntot = p["clouds"] * p["n"]
    rl = roof(Ntot, p["m"], 1) * A
    out["cfg3_reuse_loop"] = {"applications": A, "clouds": p["clouds"], "plain_ms": med,
                              "graph_ms": gmed, "graph_p10_ms": gp10, "graph_p90_ms": gp90,
                              "us_per_application_graph": gmed * 1e3 / A,
                              "strict_roofline_ms": rl, "strict_roofline_frac_graph": rl / gmed,
                              "plan_create_ms": pmed3}
    plan.close()
    del Vd, outs, g
    # eps-independence at cfg 5 (same plan re-parameterised: identical G)
    p, x, F = make_config(5)
    xd, Fd = torch.from_numpy(x).cuda(), torch.from_numpy(F).cuda()
    od = torch.empty_like(Fd)
    plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    t_a = timed(lambda: plan.integrate(Fd, out=od), 10)[0]
    plan.reparam(0.1, p["lam"])
    t_b = timed(lambda: plan.integrate(Fd, out=od), 10)[0]
    out["cfg5_eps_independence"] = {"eps_0.01_ms": t_a, "eps_0.1_ms": t_b}
    plan.reparam(p["eps"], p["lam"])
    # multi-column integrate (NEXT-2): cfg-5 points, d = 64 synthetic N(0,1)
    F64 = torch.randn((p["n"], 64), device="cuda", generator=torch.Generator("cuda").manual_seed(4))
    o64 = torch.empty_like(F64)
    t64 = timed(lambda: plan.integrate(F64, out=o64), 10)[0]
    N = p["n"]
    # NEXT-1 barycenter: k = 3 localized distributions on the cfg-5 points,
    # uniform area weights, lambda > 0 (Alg. 1 runs with lambda = 0.5 in the
    # paper); time per outer iteration (2 x 3-column integrate + 2 elementwise)
    xs = torch.from_numpy(x[:3].astype(np.float32)).cuda()
    xg = torch.from_numpy(x).cuda()
    mus = torch.exp(-((xg[None, :, :] - xs[:, None, :]) ** 2).sum(-1) / (2 * 0.25 ** 2))
    area = torch.full((p["n"],), 1.0 / p["n"], device="cuda")
    mus = (mus / (mus @ area)[:, None]).contiguous()
    try:
        plan.reparam(p["eps"], 0.01)  # lambda > 0 small enough for exp(lambda G D) in fp32
        plan.barycenter(mus, area, [1 / 3] * 3, 2)
        bts = []
        for iters in (2, 12):
            torch.cuda.synchronize()
            ev0.record(stream)
            plan.barycenter(mus, area, [1 / 3] * 3, iters)
            ev1.record(stream)
            torch.cuda.synchronize()
            bts.append(ev0.elapsed_time(ev1))
        out["cfg5_barycenter"] = {"ms_per_iteration": (bts[1] - bts[0]) / 10, "k": 3,
                                  "note": "rfd_barycenter, Alg. 1 on the cfg-5 points (N = 4M), "
                                          "k = 3, lambda = 0.01; (t(12 it) - t(2 it)) / 10"}
    except rfd.RFDError as e:  # the iteration can leave fp32 range on this cloud
        out["cfg5_barycenter"] = {"error": str(e)}
    plan.reparam(p["eps"], p["lam"])
    # NEXT-1 in the paper's regime (Table 2: meshes of 5k-19k nodes, m = 30,
    # k = 3, lambda = 0.5): the fused loop (one
    # launch, features cached on chip) vs the unfused one, per iteration
    from workloads import barycenter_inputs
    xb, ab, musb = barycenter_inputs(18944)
    pb = rfd.Plan(torch.from_numpy(xb).cuda(), 0.01, 0.5, 30, 5)  # the paper's eps, lambda, m
    mb = torch.from_numpy(musb.astype(np.float32)).cuda()
    abd = torch.from_numpy(ab.astype(np.float32)).cuda()

    def per_iter():
        ts = []
        for iters in (2, 22):
            pb.barycenter(mb, abd, [1 / 3] * 3, iters)
            torch.cuda.synchronize()
            ev0.record(stream)
            pb.barycenter(mb, abd, [1 / 3] * 3, iters)
            ev1.record(stream)
            torch.cuda.synchronize()
            ts.append(ev0.elapsed_time(ev1))
        return (ts[1] - ts[0]) / 20
    fused_ms = per_iter()
    os.environ["RFD_BARY_FUSED"] = "0"
    unfused_ms = per_iter()
    del os.environ["RFD_BARY_FUSED"]
    out["paper_barycenter"] = {"n": 18944, "m": 30, "k": 3, "eps": 0.01, "lambda": 0.5,
                               "fused_ms_per_iteration": fused_ms,
                               "unfused_ms_per_iteration": unfused_ms,
                               "note": "rfd_barycenter on 18,944 sphere points (Octocat-sized; "
                                       "synthetic bumps), (t(22 it) - t(2 it)) / 20"}
    pb.close()
    out["cfg5_d64"] = {"integrate_ms": t64, "value": N * 64 / (t64 * 1e-3), "unit": UNIT,
                       "ms_per_16_columns": t64 / 4, "d16_ms": t_a,
                       "strict_roofline_ms": roof(N, p["m"], 64),
                       "strict_roofline_frac": roof(N, p["m"], 64) / t64}
    plan.close()
    del F64, o64
    return out


def relerr(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.abs(got - ref).max() / np.abs(ref).max())


def parity_leg():
    """Max relative error (normwise, A13) of the timed workload's
    GPU result against the fp64 oracle: cfg 5 at full size, G and S over all
    4M points, out and Delta = out - F on rows at stride 1021 (every
    128-point tile lane) plus 4096 random rows and the last row."""
    import torch
    from oracle import rfd as orf
    from paper_2302_00942_b200 import rfd
    p, x, F = make_config(5)
    plan = rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
    out = plan.integrate(torch.from_numpy(F).cuda()).cpu().numpy()
    n = x.shape[0]
    rows = np.unique(np.concatenate([np.arange(0, n, 1021),
                                     np.random.default_rng(55).integers(0, n, 4096), [n - 1]]))
    t0 = time.perf_counter()
    ref = orf.Plan(x, p["eps"], p["lam"], p["m"], p["seed"])
    res = ref.apply(F, rows=rows)
    dt = time.perf_counter() - t0
    F64 = F[rows].astype(np.float64)
    errs = {"out": relerr(out[rows], res["out"]), "delta": relerr(out[rows] - F64, res["out"] - F64),
            "G": relerr(plan.export("gram"), ref.G), "C": relerr(plan.export("core"), ref.C),
            "S": relerr(plan.export("S", d=p["d"]), res["S"]),
            "Y": relerr(plan.export("Y", d=p["d"]), res["Y"])}
    plan.close()
    return {"max_rel_err_out": errs["out"], "max_rel_err_delta": errs["delta"],
            "intermediates": {k: errs[k] for k in ("G", "C", "S", "Y")}, "tolerance": 1e-4,
            "rows_compared": int(rows.size), "oracle_s": dt,
            "note": "normwise max|gpu-oracle|/max|oracle| (DESIGN.md A13) at cfg5 full size; "
                    "G and S over all N points; out / Delta on the sampled rows"}


def eps_graph_leg():
    """SURVEY 8(c) step 7 (a diagnostic, never a gate): the relative error of
    RFD (the GPU output) against the exact epsilon-graph diffusion exp(lambda A) F
    on the L-infinity (primary, reading A2) and L1 (the norm the paper names)
    graphs, cfgs 1 and 2."""
    import torch
    from oracle import dense
    from paper_2302_00942_b200 import rfd
    out = {}
    for cfg in (1, 2):
        p, x, F = make_config(cfg)
        plan = rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
        got = plan.integrate(torch.from_numpy(F).cuda()).cpu().numpy().astype(np.float64)
        plan.close()
        row = {}
        for norm, key in (("inf", "Linf"), (1, "L1")):
            ex = dense.exact_diffusion_sparse(x, F, p["eps"], p["lam"], norm)
            row["rel_err_vs_" + key] = relerr(got, ex)
            row["rel_err_delta_vs_" + key] = relerr(got - F, ex - F)
        row["m"] = p["m"]
        out["cfg%d" % cfg] = row
    out["note"] = ("approximation quality of the random-feature surrogate (m frequencies) vs the exact "
                   "graph; not a parity gate (parity is against the oracle's RF result)")
    return out


def oracle_sample(n_sample, steps=1):
    """The oracle as it stands on a bounded sample of cfg 5 (first n_sample
    points of the same generator recipe): plan + apply, all rows."""
    from oracle import rfd as orf
    p, x, F = make_config(5, n=n_sample)
    t0 = time.perf_counter()
    for _ in range(steps):
        pl = orf.Plan(x, p["eps"], p["lam"], p["m"], p["seed"])
        pl.apply(F)
    dt = (time.perf_counter() - t0) / steps
    return p, n_sample * p["d"] / dt, dt


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["rfd", "reference"], default="rfd")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=1 << 20)
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config legs")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle parity leg")
    ap.add_argument("--step-times", action="store_true",
                    help="also record an event pair per timed step and print them to stderr")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank, world, local, pg = dist_setup(args)
    p = make_config.__globals__["CONFIGS"][5]
    cfg_desc = {"workload": "cfg5_cube: N=4194304 uniform unit-cube points, m=256, d=16, "
                            "eps=0.01, lambda=-0.3 (BASELINE.json configs[4])",
                "N": p["n"], "m": p["m"], "d": p["d"], "eps": p["eps"], "lambda": p["lam"],
                "step": ("rfd_gfi (rfd_plan_create + rfd_integrate in one call; pass 1 on a second "
                         "stream beside the plan's core)" if int(os.environ.get("WORLD_SIZE", "1")) == 1
                         else "rfd_plan_create_sharded + rfd_integrate"),
                "l2": "inputs larger than L2 (F + out = 537 MB, points 67 MB per step)"}

    if args.impl == "reference":
        # The oracle (fp64 numpy) as it stands, on host cores; rank 0 only.
        if rank != 0:
            return
        ns = 65536
        for _ in range(args.warmup):
            oracle_sample(ns)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            oracle_sample(ns)
        dt = (time.perf_counter() - t0) / args.steps
        val = ns * p["d"] / dt
        line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": dict(cfg_desc, sample="first 65536 points of the cfg5 recipe per step"),
                "cpu_baseline": {"value": val, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
                                 "sample": "cfg5 recipe, N=65536 points, m=256, d=16, plan+apply"},
                "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    res = run_rfd(args, rank, world, local, pg)
    if rank != 0:
        return
    def guarded(fn, *a):
        # an optional leg that fails records its error; the bench line still prints
        try:
            return fn(*a)
        except Exception as e:  # noqa: BLE001
            return {"error": "%s: %s" % (type(e).__name__, e)}

    legs = None
    if world == 1 and not args.no_configs:
        legs = guarded(config_legs, args, peaks())
    parity = eps_graph = None
    if world == 1 and not args.no_parity:
        parity = guarded(parity_leg)
        eps_graph = guarded(eps_graph_leg)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        _, cval, cdt = oracle_sample(args.cpu_sample)
        cpu = {"value": cval, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle",
               "sample": "cfg5 recipe, first %d points, m=256, d=16, plan+apply (%.1f s)"
                         % (args.cpu_sample, cdt)}
    value = res["N"] * res["d"] * world / (res["ms_step"] * 1e-3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": dict(cfg_desc, parallelism=(
                "sharded%d: one cloud of %d x 4M points, G and S partials all-gathered over NCCL "
                "and summed in rank order (SURVEY 8(e))" % (world, world)) if world > 1 else "single GPU"),
            "roofline": res["roofline"], "cpu_baseline": cpu, "e2e": res["e2e"],
            "gpu_launches": res["launches"], "clocks": res["clocks"],
            "parity": parity, "eps_graph_diagnostic": eps_graph,
            "integrate": res["integrate"], "reparam": res["reparam"], "spectrum": res["spectrum"], "configs": legs,
            "kernels": res["kernels"],
            "gram": {"path": "spread grid (k_nufft.cu)" if res["gram_nodes"] else "direct",
                     "nodes": res["gram_nodes"],
                     "note": "a4 over a spread grid of `nodes` points (width-8 ES kernel, 8^3 taps), deconvolved "
                             "(DESIGN.md Sec. 6 'a4 spread grid'); parity as reported"}}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
