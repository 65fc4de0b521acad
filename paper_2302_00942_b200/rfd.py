"""Thin ctypes binding of the C ABI in ``include/rfd.h`` (argument marshalling only).

Every step of the method runs in the CUDA kernels of ``lib/librfd.so``; this
module only turns torch tensors / numpy arrays into pointers, streams and
sizes, and status codes into exceptions.  There is no fallback: if the
library is missing, importing the binding's entry points raises.

Names follow the ABI: ``Plan`` wraps ``rfd_plan_create`` /
``rfd_plan_create_batched`` / ``rfd_destroy``; ``Plan.sharded`` wraps
``rfd_plan_create_sharded`` (the all-gather callback is torch.distributed's
``all_gather_into_tensor``: plumbing only, the partial sums are added by the
library's kernels); ``Plan.integrate`` wraps ``rfd_integrate``;
``Plan.integrate_host`` wraps ``rfd_integrate_host``.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "librfd.so")

RFD_OK, RFD_EINVAL, RFD_ECUDA, RFD_ENOMEM, RFD_ERANGE = range(5)
RFD_MAX_M = 512
FIELDS = {"omega": 0, "nu": 1, "gram": 2, "core": 3, "S": 4, "Y": 5}

# Every symbol include/rfd.h declares (checked by tests/test_abi.py).
EXPORTED = ("rfd_plan_create", "rfd_plan_create_batched", "rfd_plan_create_sharded",
            "rfd_plan_reparam",
            "rfd_plan_spectrum", "rfd_barycenter", "rfd_integrate",
            "rfd_integrate_host", "rfd_gfi", "rfd_gfi_host", "rfd_destroy", "rfd_last_error",
            "rfd_plan_info",
            "rfd_plan_export", "rfd_launch_count", "rfd_profile_enable",
            "rfd_profile_only", "rfd_profile_read")


class RFDError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("rfd status %d: %s" % (status, msg))
        self.status = status


class PlanInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("batch", ctypes.c_int32), ("m", ctypes.c_int32),
                ("r", ctypes.c_int32), ("scaling", ctypes.c_int32),
                ("symmetric", ctypes.c_int32), ("eps", ctypes.c_double),
                ("lam", ctypes.c_double), ("seed", ctypes.c_uint64),
                ("n_total", ctypes.c_int64), ("rank", ctypes.c_int32),
                ("world", ctypes.c_int32), ("gram_nodes", ctypes.c_int64)]


# int allgather(void* ctx, const double* send, double* recv, size_t count, stream)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_size_t, ctypes.c_void_p)


class Shard(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("allgather", ALLGATHER_FN), ("ctx", ctypes.c_void_p)]


def shard_rows(n, rank, world):
    """Contiguous partition of n points over `world` ranks: rank q owns rows
    [n q / world, n (q + 1) / world) (sizes differ by at most one)."""
    return (n * rank) // world, (n * (rank + 1)) // world


class _DeviceArray:
    """A raw fp64 buffer as a tensor view (__cuda_array_interface__)."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3}


def _view(ptr, count, device):
    import torch
    if device.type == "cuda":
        return torch.as_tensor(_DeviceArray(ptr, count), device=device)
    buf = (ctypes.c_double * int(count)).from_address(int(ptr))
    return torch.frombuffer(buf, dtype=torch.float64)


def make_allgather(group=None, device=None):
    """The rfd_allgather_fn for a torch.distributed process group: wraps the
    library's send / recv buffers (device pointers; host pointers when
    ``device`` is the CPU -- gloo, tests) and all-gathers rank-major, ordered
    on the library's stream.  Returns the ctypes callback (keep a reference)."""
    import torch
    import torch.distributed as dist
    dev = torch.device(device if device is not None else "cuda")
    world = dist.get_world_size(group)

    def cb(_ctx, send, recv, count, stream):
        try:
            src = _view(send, count, dev)
            dst = _view(recv, count * world, dev)
            if dev.type == "cuda":
                with torch.cuda.stream(torch.cuda.ExternalStream(int(stream or 0), device=dev)):
                    dist.all_gather_into_tensor(dst, src, group=group)
            else:
                dist.all_gather(list(dst.view(world, int(count)).unbind(0)), src, group=group)
            return 0
        except Exception as e:  # no exception may cross the C ABI
            import sys
            print("rfd allgather failed: %r" % (e,), file=sys.stderr)
            return 1
    return ALLGATHER_FN(cb)


class ProfileEntry(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 48), ("launches", ctypes.c_int64),
                ("total_ms", ctypes.c_double)]


_lib = None


def load_library(path=LIB_PATH):
    """Load librfd.so (raises if it has not been built: no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError("librfd.so not built at %s; run `python -m "
                           "paper_2302_00942_b200.build` (there is no CPU fallback)" % path)
    lib = ctypes.CDLL(path)
    vp, i64, i32, dbl, u64 = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                              ctypes.c_double, ctypes.c_uint64)
    pp = ctypes.POINTER(ctypes.c_void_p)
    lib.rfd_plan_create.argtypes = [vp, i64, dbl, dbl, i32, u64, vp, pp]
    lib.rfd_plan_create_batched.argtypes = [vp, i32, i64, dbl, dbl, i32, u64, vp, pp]
    lib.rfd_plan_create_sharded.argtypes = [vp, i64, dbl, dbl, i32, u64, ctypes.POINTER(Shard),
                                            vp, pp]
    lib.rfd_plan_reparam.argtypes = [vp, dbl, dbl, vp]
    lib.rfd_plan_spectrum.argtypes = [vp, i32, vp, vp]
    lib.rfd_barycenter.argtypes = [vp, vp, vp, vp, i32, i32, dbl, vp, ctypes.POINTER(i32), vp]
    lib.rfd_integrate.argtypes = [vp, vp, i32, vp, vp]
    lib.rfd_integrate_host.argtypes = [vp, vp, i32, vp, vp]
    lib.rfd_gfi_host.argtypes = [vp, i64, dbl, dbl, i32, u64, vp, i32, vp, vp, pp]
    lib.rfd_gfi.argtypes = [vp, i64, dbl, dbl, i32, u64, vp, i32, vp, vp, pp]
    lib.rfd_destroy.argtypes = [vp]
    lib.rfd_destroy.restype = None
    lib.rfd_last_error.restype = ctypes.c_char_p
    lib.rfd_plan_info.argtypes = [vp, ctypes.POINTER(PlanInfo)]
    lib.rfd_plan_export.argtypes = [vp, ctypes.c_int, vp, ctypes.c_size_t]
    lib.rfd_launch_count.restype = ctypes.c_uint64
    lib.rfd_profile_enable.argtypes = [ctypes.c_int]
    lib.rfd_profile_only.argtypes = [ctypes.c_char_p]
    lib.rfd_profile_read.argtypes = [ctypes.POINTER(ProfileEntry), i32]
    lib.rfd_profile_read.restype = i32
    for name in ("rfd_plan_create", "rfd_plan_create_batched", "rfd_plan_create_sharded",
                 "rfd_plan_reparam",
                 "rfd_plan_spectrum", "rfd_barycenter", "rfd_integrate",
                 "rfd_integrate_host", "rfd_gfi", "rfd_gfi_host", "rfd_plan_info", "rfd_plan_export",
                 "rfd_profile_enable", "rfd_profile_only"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(status):
    if status != RFD_OK:
        raise RFDError(status, load_library().rfd_last_error().decode())


def _stream_handle(stream, device=None):
    import torch
    if stream is None:
        # the current stream's raw handle without building a Stream object
        # (the per-call host cost bounds the small configurations' plain loop)
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        if raw is not None:
            return ctypes.c_void_p(raw(torch.cuda.current_device() if device is None else device))
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(a):
    """Data pointer of a contiguous torch tensor or numpy array."""
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return ctypes.c_void_p(a.ctypes.data)
    if not a.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return ctypes.c_void_p(a.data_ptr())


def _check_f32(a, name):
    if isinstance(a, np.ndarray):
        ok = a.dtype == np.float32
    else:
        import torch
        ok = a.dtype is torch.float32
    if not ok:
        raise TypeError("%s must be float32" % name)


class Plan:
    """An RFD plan: omega, nu, G and the core C^ for one cloud or a batch.

    ``points``: (N, 3) or, batched, (B, N, 3) float32 -- a CUDA tensor or a
    host tensor / numpy array (the library copies it).
    """

    def __init__(self, points, eps, lam, m, seed, stream=None, _shard=None):
        lib = load_library()
        _check_f32(points, "points")
        shape = tuple(points.shape)
        self._keep = points
        self._shard = _shard  # (keeps the allgather callback alive)
        handle = ctypes.c_void_p()
        s = _stream_handle(stream)
        if _shard is not None:
            if len(shape) != 2 or shape[1] != 3:
                raise ValueError("a shard's points must be (n_local, 3)")
            self.batch, self.n = 1, shape[0]
            st = lib.rfd_plan_create_sharded(_ptr(points), self.n, float(eps), float(lam), int(m),
                                             int(seed), ctypes.byref(_shard), s,
                                             ctypes.byref(handle))
        elif len(shape) == 2 and shape[1] == 3:
            self.batch, self.n = 1, shape[0]
            st = lib.rfd_plan_create(_ptr(points), self.n, float(eps), float(lam), int(m),
                                     int(seed), s, ctypes.byref(handle))
        elif len(shape) == 3 and shape[2] == 3:
            self.batch, self.n = shape[0], shape[1]
            st = lib.rfd_plan_create_batched(_ptr(points), self.batch, self.n, float(eps),
                                             float(lam), int(m), int(seed), s,
                                             ctypes.byref(handle))
        else:
            raise ValueError("points must be (N, 3) or (B, N, 3)")
        _check(st)
        self._h = handle
        self.m, self.r = int(m), 2 * int(m)
        self.eps, self.lam, self.seed = float(eps), float(lam), int(seed)
        self._keep = None

    @classmethod
    def sharded(cls, points_local, eps, lam, m, seed, group=None, stream=None):
        """This rank's shard (n_local x 3 CUDA points) of one cloud split over
        the ranks of a torch.distributed process group: the
        Gram and S partials are all-gathered and summed in rank order by the
        library; every rank gets the same C^ and its own rows of out."""
        import torch.distributed as dist
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        import torch
        # the library's send / recv buffers are device memory (points may be host)
        dev = torch.device("cuda", torch.cuda.current_device())
        cb = make_allgather(group, dev) if world > 1 else ALLGATHER_FN()
        shard = Shard(rank, world, cb, None)
        return cls(points_local, eps, lam, m, seed, stream=stream, _shard=shard)

    # -- lifecycle ---------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            load_library().rfd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def reparam(self, eps, lam, stream=None):
        """New (eps, lambda) on the stored Gram matrix: nu and C^ only (NEXT-4)."""
        _check(load_library().rfd_plan_reparam(self._h, float(eps), float(lam),
                                               _stream_handle(stream)))
        self.eps, self.lam = float(eps), float(lam)
        return self

    def spectrum(self, k, stream=None):
        """k smallest eigenvalues of exp(lambda W~) per cloud (NEXT-3), numpy fp64
        of shape (k,) or (B, k)."""
        out = np.empty((self.batch, max(int(k), 1)), np.float64)  # k < 1: the ABI rejects it
        _check(load_library().rfd_plan_spectrum(self._h, int(k), _ptr(out),
                                                _stream_handle(stream)))
        return out[0] if self.batch == 1 else out

    def barycenter(self, mus, area, alpha, max_iter, tol=0.0, stream=None):
        """Wasserstein barycenter (Alg. 1, NEXT-1) of the k rows of ``mus``
        (CUDA float32 k x N) with area weights ``area`` (CUDA float32 N).
        Returns (mu CUDA float32 N, iterations run)."""
        import torch
        _check_f32(mus, "mus")
        _check_f32(area, "area")
        # the kernels read k x N and N elements: undersized buffers would be
        # read out of bounds, so the shapes are checked here
        if mus.dim() != 2 or int(mus.shape[1]) != self.n:
            raise ValueError("mus must be (k, %d)" % self.n)
        if area.numel() != self.n:
            raise ValueError("area must have %d elements" % self.n)
        if not (mus.is_cuda and area.is_cuda) or mus.device != area.device:
            raise ValueError("mus and area must be CUDA tensors on the plan's device")
        k = int(mus.shape[0])
        al = np.ascontiguousarray(np.asarray(alpha, np.float64))
        out = torch.empty((self.n,), dtype=torch.float32, device=mus.device)
        its = ctypes.c_int32(0)
        _check(load_library().rfd_barycenter(self._h, _ptr(mus), _ptr(area), _ptr(al), k,
                                             int(max_iter), float(tol), _ptr(out),
                                             ctypes.byref(its), _stream_handle(stream)))
        return out, its.value

    # -- inference -----------------------------------------------------------
    def _field_dims(self, F):
        shape = tuple(F.shape)
        lead = (self.batch, self.n) if self.batch > 1 else (self.n,)
        if shape[:len(lead)] != lead or len(shape) > len(lead) + 1:
            raise ValueError("F must have shape %s or %s + (d,)" % (lead, lead))
        return 1 if len(shape) == len(lead) else shape[-1]

    def integrate(self, F, out=None, stream=None):
        """out = exp(lambda W~) F for a CUDA float32 tensor F ((B,) N[, d]).

        ``out`` may be F itself (in place).  Asynchronous on ``stream``.
        """
        import torch
        _check_f32(F, "F")
        if not F.is_cuda:
            raise ValueError("F must be a CUDA tensor (use integrate_host for host buffers)")
        d = self._field_dims(F)
        if out is None:
            out = torch.empty_like(F)
        elif out.shape != F.shape or not out.is_cuda:
            raise ValueError("out must be a CUDA tensor shaped like F")
        else:
            _check_f32(out, "out")
        _check(load_library().rfd_integrate(self._h, _ptr(F), d, _ptr(out),
                                            _stream_handle(stream, F.device.index)))
        return out

    def integrate_host(self, F_host, out_host, stream=None):
        """Same with HOST buffers (pinned for asynchrony): H2D, integrate, D2H."""
        _check_f32(F_host, "F")
        _check_f32(out_host, "out")
        d = self._field_dims(F_host)
        if tuple(out_host.shape) != tuple(F_host.shape):
            raise ValueError("out must be shaped like F")
        _check(load_library().rfd_integrate_host(self._h, _ptr(F_host), d, _ptr(out_host),
                                                 _stream_handle(stream)))
        return out_host

    # -- introspection -------------------------------------------------------
    def info(self):
        inf = PlanInfo()
        _check(load_library().rfd_plan_info(self._h, ctypes.byref(inf)))
        return {f: getattr(inf, f) for f, _ in PlanInfo._fields_}

    def export(self, field, d=None):
        """Copy plan state to host numpy (paper's [cos; sin] feature order)."""
        B, m, r = self.batch, self.m, self.r
        if field == "omega":
            arr = np.empty((m, 3), np.float32)
        elif field == "nu":
            arr = np.empty((m,), np.float64)
        elif field in ("gram", "core"):
            arr = np.empty((B, r, r), np.float64)
        elif field in ("S", "Y"):
            if d is None:
                raise ValueError("pass d (the d of the last integrate)")
            arr = np.empty((B, r, d), np.float64 if field == "S" else np.float32)
        else:
            raise ValueError("unknown field %r" % field)
        _check(load_library().rfd_plan_export(self._h, FIELDS[field], _ptr(arr), arr.nbytes))
        if field in ("gram", "core", "S", "Y") and B == 1:
            arr = arr[0]
        return arr


def _plan_from_handle(handle, n, eps, lam, m, seed):
    plan = Plan.__new__(Plan)
    plan._h, plan._keep, plan._shard = handle, None, None
    plan.batch, plan.n, plan.m, plan.r = 1, n, int(m), 2 * int(m)
    plan.eps, plan.lam, plan.seed = float(eps), float(lam), int(seed)
    return plan


def gfi(points, eps, lam, m, seed, F, out=None, keep_plan=False, stream=None):
    """rfd_gfi: plan + integrate of a DEVICE field in one call (pass 1 beside
    the plan's core).  points (N, 3) float32 (host or device); F (N[, d])
    float32 on the GPU; out like F (allocated when None).  Returns out, or
    (out, Plan) when keep_plan."""
    import torch
    lib = load_library()
    _check_f32(points, "points")
    _check_f32(F, "F")
    n = int(points.shape[0])
    if tuple(points.shape) != (n, 3) or int(F.shape[0]) != n:
        raise ValueError("points (N, 3) and F (N[, d]) expected")
    if out is None:
        out = torch.empty_like(F)
    _check_f32(out, "out")
    if tuple(out.shape) != tuple(F.shape):
        raise ValueError("out must have F's shape")
    d = 1 if len(F.shape) == 1 else int(F.shape[1])
    handle = ctypes.c_void_p()
    _check(lib.rfd_gfi(_ptr(points), n, float(eps), float(lam), int(m), int(seed), _ptr(F), d,
                       _ptr(out), _stream_handle(stream),
                       ctypes.byref(handle) if keep_plan else None))
    if not keep_plan:
        return out
    return out, _plan_from_handle(handle, n, eps, lam, m, seed)


def gfi_host(points, eps, lam, m, seed, F_host, out_host, keep_plan=False, stream=None):
    """rfd_gfi_host: plan + integrate from HOST buffers in one call, the
    transfers overlapped with the computation.  points (N, 3), F_host and
    out_host (N[, d]) host float32 (pinned for asynchrony).  Returns the Plan
    when keep_plan, else None; synchronize the stream before reading out_host."""
    lib = load_library()
    for a, nm in ((points, "points"), (F_host, "F"), (out_host, "out")):
        _check_f32(a, nm)
    n = int(points.shape[0])
    if tuple(points.shape) != (n, 3) or int(F_host.shape[0]) != n or \
            tuple(out_host.shape) != tuple(F_host.shape):
        raise ValueError("points (N, 3), F and out (N[, d]) expected")
    d = 1 if len(F_host.shape) == 1 else int(F_host.shape[1])
    handle = ctypes.c_void_p()
    _check(lib.rfd_gfi_host(_ptr(points), n, float(eps), float(lam), int(m), int(seed),
                            _ptr(F_host), d, _ptr(out_host), _stream_handle(stream),
                            ctypes.byref(handle) if keep_plan else None))
    if not keep_plan:
        return None
    return _plan_from_handle(handle, n, eps, lam, m, seed)


def launch_count():
    return int(load_library().rfd_launch_count())


def profile_enable(on=True):
    _check(load_library().rfd_profile_enable(1 if on else 0))


def profile_only(name=None):
    """Profile only launches named `name` (None: every launch)."""
    _check(load_library().rfd_profile_only(name.encode() if name else None))


def profile_read(cap=64):
    """{kernel name: (launches, total_ms)} since the last enable/read (synchronizes)."""
    arr = (ProfileEntry * cap)()
    k = load_library().rfd_profile_read(arr, cap)
    return {arr[i].name.decode(): (int(arr[i].launches), float(arr[i].total_ms)) for i in range(k)}
