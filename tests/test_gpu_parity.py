"""CUDA path vs the fp64 oracle, through the C ABI (needs a B200).

Tolerance (BASELINE.json north star; A13): normwise
    max_{i,c} |out_gpu - out_ref| / max_{i,c} |out_ref| <= 1e-4,
and the same gate on the correction Delta = out - F, which is only 0.5-1.2 %
of max|out| on the random-field configs and would otherwise be invisible.
Intermediates (G, C^, S, Y) are compared normwise against their own max-abs.
omega is compared bit for bit (the stream is part of the contract, A14).
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import rfd as orf  # noqa: E402
from paper_2302_00942_b200 import rfd  # noqa: E402
from workloads import make_config  # noqa: E402

TOL = 1e-4


def relerr(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.abs(got - ref).max() / np.abs(ref).max())


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rfd.load_library()


def _run_single(x, F, p):
    xd = torch.from_numpy(x).cuda()
    Fd = torch.from_numpy(np.ascontiguousarray(F)).cuda()
    plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    out = plan.integrate(Fd).cpu().numpy()
    return plan, out


def _check_against_oracle(plan, out, x, F, p, rows=None, d=None):
    ref = orf.Plan(x, p["eps"], p["lam"], p["m"], p["seed"])
    omega = plan.export("omega")
    np.testing.assert_array_equal(omega, ref.omega)
    np.testing.assert_allclose(plan.export("nu"), ref.nu, rtol=1e-12)
    errs = {"G": relerr(plan.export("gram"), ref.G), "C": relerr(plan.export("core"), ref.C)}
    res = ref.apply(F, rows=rows)
    d = F.reshape(F.shape[0], -1).shape[1]
    errs["S"] = relerr(plan.export("S", d=d), res["S"])
    errs["Y"] = relerr(plan.export("Y", d=d), res["Y"])
    F2 = F.reshape(F.shape[0], -1).astype(np.float64)
    o2 = out.reshape(out.shape[0], -1)
    if rows is not None:
        F2, o2 = F2[rows], o2[rows]
    errs["out"] = relerr(o2, res["out"])
    errs["delta"] = relerr(o2 - F2, res["out"] - F2)
    print(p["name"], {k: "%.2e" % v for k, v in errs.items()})
    for k, v in errs.items():
        assert v <= TOL, (k, v)
    return errs


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_config_parity(cfg):
    p, x, F = make_config(cfg)
    plan, out = _run_single(x, F, p)
    _check_against_oracle(plan, out, x, F, p)


@pytest.mark.slow
def test_config5_full_size_parity():
    # Full N = 4M, m = 256, d = 16, in the launch configuration bench.py times;
    # out compared on 4096 sampled rows (every row still enters G and S).
    p, x, F = make_config(5)
    plan, out = _run_single(x, F, p)
    # rows at a prime stride (1021: every residue mod 128, i.e. every lane of
    # the 128-point pass-2 tiles and every 16-point group position) plus 4096
    # random rows and the last row
    n = x.shape[0]
    rng = np.random.default_rng(55)
    rows = np.unique(np.concatenate([np.arange(0, n, 1021), rng.integers(0, n, 4096), [n - 1]]))
    assert len(np.unique(rows % 128)) == 128
    _check_against_oracle(plan, out, x, F, p, rows=rows)


def test_config3_batched_fifty_applications():
    p, x, V = make_config(3)
    B, n, A = p["clouds"], p["n"], p["applications"]
    xd = torch.from_numpy(x).cuda()
    plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    Vd = torch.from_numpy(V).cuda()  # (A, B, n, 1)
    outs = torch.empty_like(Vd)
    for t in range(A):
        plan.integrate(Vd[t], out=outs[t])
    outs = outs.cpu().numpy()
    G = plan.export("gram")
    C = plan.export("core")
    worst = {"out": 0.0, "delta": 0.0, "G": 0.0, "C": 0.0}
    for b in range(B):
        ref = orf.Plan(x[b], p["eps"], p["lam"], p["m"], p["seed"])
        # The integrator is linear in F: the 50 applications of cloud b are the
        # 50 columns of one oracle apply.
        Fb = V[:, b, :, 0].T.astype(np.float64)
        res = ref.apply(Fb)
        ob = outs[:, b, :, 0].T
        for t in range(A):
            worst["out"] = max(worst["out"], relerr(ob[:, t], res["out"][:, t]))
            worst["delta"] = max(worst["delta"], relerr(ob[:, t] - Fb[:, t], res["out"][:, t] - Fb[:, t]))
        worst["G"] = max(worst["G"], relerr(G[b], ref.G))
        worst["C"] = max(worst["C"], relerr(C[b], ref.C))
    print("cfg3", {k: "%.2e" % v for k, v in worst.items()})
    for k, v in worst.items():
        assert v <= TOL, (k, v)


def test_omega_bitwise_all_seeds():
    for cfg in (1, 2, 3, 4, 5):
        p, x, _ = make_config(cfg) if cfg != 5 else make_config(5, n=1024)
        xs = x.reshape(-1, 3)[:64].copy()
        plan = rfd.Plan(torch.from_numpy(xs).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
        om, _ = orf.frequencies(p["seed"], p["m"])
        np.testing.assert_array_equal(plan.export("omega"), om)
        assert plan.info()["symmetric"] == 1


# ---------------------------------------------------------------- edge cases
def _sphere(n, seed):
    g = np.random.default_rng(seed).standard_normal((n, 3))
    return (g / np.linalg.norm(g, axis=1, keepdims=True)).astype(np.float32)


@pytest.mark.parametrize("n,m,d", [(1, 16, 3), (2, 8, 1), (37, 1, 2), (1000, 40, 5),
                                   (4099, 33, 20), (3001, 512, 4), (70001, 96, 37),
                                   (12345, 128, 16)])
def test_ragged_shapes_parity(n, m, d):
    # eps = 0.05 keeps every sinc factor in its first lobe (all nu > 0:
    # symmetric core route).
    x = _sphere(n, n + m)
    F = np.random.default_rng(d).standard_normal((n, d)).astype(np.float32)
    p = dict(name="ragged n=%d m=%d d=%d" % (n, m, d), eps=0.05, lam=-0.8, m=m, seed=11)
    plan, out = _run_single(x, F, p)
    assert plan.info()["symmetric"] == 1
    _check_against_oracle(plan, out, x, F, p)


def test_field_column_scales_parity():
    # Pass 1 scales each channel of F by a power of two into fp16 range
    # (pass 1): columns spanning 1e-30 .. 1e30, a zero column and
    # a column with one nonzero entry must each meet the tolerance on their own.
    n, m = 3000, 64
    x = _sphere(n, 5)
    g = np.random.default_rng(6).standard_normal((n, 6))
    scales = np.array([1e-30, 1e-6, 1.0, 1e6, 1e30, 0.0])
    F = (g * scales).astype(np.float32)
    F[:, 5] = 0.0
    F[1234, 5] = 3.0
    p = dict(name="column scales", eps=0.05, lam=-0.8, m=m, seed=21)
    plan, out = _run_single(x, F, p)
    ref = orf.Plan(x, p["eps"], p["lam"], p["m"], p["seed"]).apply(F.astype(np.float64))
    for c in range(6):
        e_out = relerr(out[:, c], ref["out"][:, c])
        e_del = relerr(out[:, c] - F[:, c].astype(np.float64), ref["out"][:, c] - F[:, c])
        print("column", c, "%.2e %.2e" % (e_out, e_del))
        assert e_out <= TOL and e_del <= TOL, (c, e_out, e_del)


@pytest.mark.parametrize("shift,scale", [(10.0, 1.0), (100.0, 1.0), (1000.0, 1.0), (0.0, 50.0),
                                         (0.0, 10.0)])
def test_translated_and_scaled_clouds_parity(shift, scale):
    # W depends on n_i - n_j only (Eq. 9): the exact result
    # is translation-invariant.  The library centres every cloud on its
    # bounding box (k_freq.cu) and rotates the exported G, C^, S, Y back, so a
    # translated cloud meets the gate like the original; the fp32 feature
    # argument's error grows with |omega|_1 * half-extent (scaled clouds,
    # include/rfd.h "Coordinate range").
    p, x, F = make_config(2)
    x = (x.astype(np.float64) * scale + shift * np.array([1.0, -0.7, 0.4])).astype(np.float32)
    p = dict(p, name="cfg2 shift %g scale %g" % (shift, scale))
    plan, out = _run_single(x, F, p)
    _check_against_oracle(plan, out, x, F, p)


def test_permutation_equivariance():
    # K = exp(lambda W~) with W~ = Phi D Phi^T: permuting the points permutes
    # rows and columns of K: out(P x, P F) = P out(x, F)
    # (sums over points in another order: fp32 rounding only).
    p, x, F = make_config(2)
    perm = np.random.default_rng(8).permutation(x.shape[0])
    _, out = _run_single(x, F, p)
    _, outp = _run_single(np.ascontiguousarray(x[perm]), np.ascontiguousarray(F[perm]), p)
    assert relerr(outp, out[perm]) <= 1e-5
    assert relerr(outp - F[perm], out[perm] - F[perm]) <= 1e-5


def test_tiny_field_columns_pass2_scale_clamp():
    # Pass 2 scales Y per channel by 2^(14 - e) into fp16 range; for max|Y_j|
    # below 2^-113 (a field column ~1e-33, or a tiny lambda) the scale is
    # clamped at 2^126 instead of overflowing to inf and turning the column
    # into NaN.  Columns of ~1e-33 and ~1e-36 (fp32 normal) must
    # still meet the gates on out and on Delta.
    n, m = 3000, 64
    x = _sphere(n, 5)
    # (d = 5: the tensor-core passes; d <= 4 runs the one-launch SIMT path)
    F = np.random.default_rng(7).standard_normal((n, 5)).astype(np.float32)
    F[:, 1] *= np.float32(1e-33)
    F[:, 2] *= np.float32(1e-36)
    p = dict(name="tiny columns", eps=0.05, lam=-0.8, m=m, seed=21)
    res = orf.Plan(x, p["eps"], p["lam"], p["m"], p["seed"]).apply(F.astype(np.float64))
    assert np.abs(res["Y"][:, 1]).max() < 2.0 ** -113  # the clamped branch is exercised
    plan, out = _run_single(x, F, p)
    assert np.isfinite(out).all()
    for c in range(5):
        e_out = relerr(out[:, c], res["out"][:, c])
        e_del = relerr(out[:, c] - F[:, c].astype(np.float64), res["out"][:, c] - F[:, c])
        print("tiny column", c, "%.2e %.2e" % (e_out, e_del))
        assert e_out <= TOL and e_del <= TOL, (c, e_out, e_del)


def test_misaligned_field_rejected():
    # include/rfd.h: F and out must be 16-byte aligned (pass 1 bulk-copies
    # F blocks, pass 2 uses 16-byte loads and stores): EINVAL otherwise, and
    # the plan stays usable.
    n, d = 3001, 16
    x = _sphere(n, 17)
    F = np.random.default_rng(3).standard_normal((n, d)).astype(np.float32)
    plan = rfd.Plan(torch.from_numpy(x).cuda(), 0.05, -0.8, 128, 9)
    Fd = torch.from_numpy(F).cuda()
    buf = torch.empty(n * d + 1, device="cuda")
    Fu = buf[1:].view(n, d)
    assert Fu.data_ptr() % 16 == 4
    Fu.copy_(Fd)
    with pytest.raises(rfd.RFDError, match="aligned"):
        plan.integrate(Fu)
    with pytest.raises(rfd.RFDError, match="aligned"):
        plan.integrate(Fd, out=torch.empty(n * d + 1, device="cuda")[1:].view(n, d))
    out = plan.integrate(Fd).cpu().numpy()
    oref = orf.Plan(x, 0.05, -0.8, 128, 9).apply(F.astype(np.float64))["out"]
    assert relerr(out, oref) <= TOL


@pytest.mark.parametrize("cfg", [2, 4])
def test_reparam_bitwise_equals_fresh_plan_and_oracle(cfg):
    # NEXT-4: rfd_plan_reparam keeps G and recomputes nu and C^; the result is
    # bit-identical to a fresh plan (same kernels, same inputs) and meets the
    # oracle at the new parameters.
    p, x, F = make_config(cfg)
    xd, Fd = torch.from_numpy(x).cuda(), torch.from_numpy(F).cuda()
    eps2, lam2 = p["eps"] * 1.5, p["lam"] * 0.5
    plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    G0 = plan.export("gram")
    plan.reparam(eps2, lam2)
    fresh = rfd.Plan(xd, eps2, lam2, p["m"], p["seed"])
    np.testing.assert_array_equal(plan.export("gram"), G0)
    np.testing.assert_array_equal(plan.export("gram"), fresh.export("gram"))
    np.testing.assert_array_equal(plan.export("nu"), fresh.export("nu"))
    np.testing.assert_array_equal(plan.export("core"), fresh.export("core"))
    assert plan.info()["eps"] == eps2 and plan.info()["lam"] == lam2
    assert plan.info()["scaling"] == fresh.info()["scaling"]
    out = plan.integrate(Fd).cpu().numpy()
    np.testing.assert_array_equal(out, fresh.integrate(Fd).cpu().numpy())
    q = dict(p, eps=eps2, lam=lam2, name="reparam cfg%d" % cfg)
    _check_against_oracle(plan, out, x, F, q)


def test_reparam_errors_leave_plan_unchanged():
    p, x, F = make_config(1)
    xd, Fd = torch.from_numpy(x).cuda(), torch.from_numpy(F).cuda()
    plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    before = plan.integrate(Fd).cpu().numpy()
    C0 = plan.export("core")
    for eps, lam in [(0.0, -0.5), (-1.0, -0.5), (float("nan"), -0.5), (0.1, float("inf"))]:
        with pytest.raises(rfd.RFDError):
            plan.reparam(eps, lam)
    # overflow (large lambda > 0): ERANGE, plan unchanged
    with pytest.raises(rfd.RFDError):
        plan.reparam(p["eps"], 1e6)
    np.testing.assert_array_equal(plan.export("core"), C0)
    assert plan.info()["lam"] == p["lam"]
    np.testing.assert_array_equal(plan.integrate(Fd).cpu().numpy(), before)


@pytest.mark.parametrize("cfg,k", [(1, 32), (2, 64), (4, 200), (1, 1024)])
def test_spectrum_matches_oracle(cfg, k):
    # NEXT-3: k smallest eigenvalues of exp(lambda W~) (GPU: Householder
    # tridiagonalisation of D^1/2 G D^1/2 + bisection; oracle: general
    # eigenvalues of its own G D).  Values lie in (0, 1] for lambda < 0;
    # gate 1e-4 absolute (the G parity gate carried through exp).
    p, x, F = make_config(cfg)
    plan = rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
    got = plan.spectrum(k)
    ref = orf.Plan(x, p["eps"], p["lam"], p["m"], p["seed"]).spectrum(k)
    err = float(np.abs(got - ref).max())
    print("spectrum cfg%d k=%d max abs err %.2e" % (cfg, k, err))
    assert got.shape == (k,)
    assert np.all(np.diff(got) >= 0)
    assert err <= 1e-4


def test_spectrum_batched_and_small_clouds():
    # cfg-3-like batch (r = 64 per cloud) and clouds with N < r.
    rng = np.random.default_rng(3)
    for n, m, B in [(300, 32, 8), (20, 16, 3)]:
        x = rng.random((B, n, 3), dtype=np.float32)
        plan = rfd.Plan(torch.from_numpy(x).cuda(), 0.1, -2.0, m, 5)
        k = min(n, 16)
        got = plan.spectrum(k)
        assert got.shape == (B, k)
        for b in range(B):
            ref = orf.Plan(x[b], 0.1, -2.0, m, 5).spectrum(k)
            assert float(np.abs(got[b] - ref).max()) <= 1e-4, (n, m, b)


def test_spectrum_errors():
    p, x, F = make_config(1)
    plan = rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
    for k in (0, -1, x.shape[0] + 1):
        with pytest.raises(rfd.RFDError):
            plan.spectrum(k)


@pytest.mark.parametrize("n,m,d", [(20000, 256, 64), (9001, 256, 100), (6000, 512, 50),
                                   (5000, 64, 33)])
def test_multi_column_parity(n, m, d):
    # NEXT-2: pass 2 takes up to 64 columns per launch (MMA N = the chunk's
    # columns, Y^T scaled per channel); wide and ragged d against the oracle.
    x = _sphere(n, n + d)
    F = np.random.default_rng(d).standard_normal((n, d)).astype(np.float32)
    F[:, -1] *= 1e3  # channels of very different scales in one chunk
    p = dict(name="multicol n=%d m=%d d=%d" % (n, m, d), eps=0.05, lam=-0.8, m=m, seed=17)
    plan, out = _run_single(x, F, p)
    _check_against_oracle(plan, out, x, F, p)


def _bary_gpu(plan, mus, a, alpha, iters, tol=0.0):
    mus_d = torch.from_numpy(np.ascontiguousarray(mus, dtype=np.float32)).cuda()
    a_d = torch.from_numpy(a.astype(np.float32)).cuda()
    got, its = plan.barycenter(mus_d, a_d, alpha, iters, tol=tol)
    return got.cpu().numpy().astype(np.float64), its


def _bary_hybrid(plan, mus, a, alpha, iters, tol=0.0):
    """Alg. 1 in fp64 numpy with FM_K = the GPU integrate, its inputs formed
    exactly as k_sinkhorn.cu forms them (X = fp32(a v s), s = 2^-e of the
    column max of a v; FM_K(a v) = Y / s).  Same FM_K arithmetic, so it
    reproduces rfd_barycenter up to fp64 rounding of the elementwise steps."""
    a32 = a.astype(np.float32).astype(np.float64)
    Mt = np.ascontiguousarray(mus.astype(np.float32).T).astype(np.float64)
    n, k = Mt.shape
    al = np.asarray(alpha, np.float64)

    def fm(Z):
        col = (a32[:, None] * Z).max(axis=0)
        s = np.array([2.0 ** -np.frexp(c)[1] if c > 0 else 1.0 for c in col])
        X = ((a32[:, None] * Z) * s[None, :]).astype(np.float32)
        Y = plan.integrate(torch.from_numpy(X).cuda()).cpu().numpy().astype(np.float64)
        return Y / s[None, :]

    V = np.ones((n, k))
    mu = np.ones(n)
    it = 0
    for it in range(1, iters + 1):
        mu_old = mu
        W = Mt / np.maximum(fm(V), 1e-30)
        d = np.maximum(V * fm(W), 1e-30)
        lg = np.zeros(n)
        for i in range(k):
            lg = lg + al[i] * np.log(d[:, i])
        mu = np.exp(lg)
        V = (V * mu[:, None]) / d
        if tol > 0 and np.abs(mu - mu_old).sum() < tol:
            break
    return mu / float(a32 @ mu), it


def test_barycenter_identity_kernel_closed_form():
    # NEXT-1 with FM = identity (lambda = 0: the integrate returns F exactly):
    # every iteration gives the weighted geometric mean prod_i (mu^i)^alpha_i
    # normalised to <a, mu> = 1 (Alg. 1 step 3, PAPER.md:1046;
    # tests/test_oracle_integrator.py::test_barycenter_geometric_mean_pin).
    from workloads import barycenter_inputs

    x, a, mus = barycenter_inputs(3000, floor=0.05, k=3)
    a = np.random.default_rng(3).uniform(0.5, 1.5, a.shape)
    a /= a.sum()
    mus = mus / (mus @ a)[:, None]
    plan = rfd.Plan(torch.from_numpy(x).cuda(), 0.05, 0.0, 64, 5)
    m32 = mus.astype(np.float32).astype(np.float64)
    a32 = a.astype(np.float32).astype(np.float64)
    for alpha in ([0.25, 0.75], [1 / 3] * 3):
        k = len(alpha)
        geo = np.prod(m32[:k] ** np.asarray(alpha)[:, None], axis=0)
        geo /= a32 @ geo
        for iters in (1, 10):
            got, its = _bary_gpu(plan, mus[:k], a, alpha, iters)
            assert its == iters
            assert relerr(got, geo) <= 1e-6, (alpha, iters, relerr(got, geo))
        # fixed point at iteration 1 (up to the fp32 rounding of FM_K's input,
        # ~1e-7 of each mu_n: sum |mu_2 - mu_1| ~ 3e-4)
        _, its = _bary_gpu(plan, mus[:k], a, alpha, 50, tol=1e-3)
        assert its == 2


@pytest.mark.parametrize("floor", [0.0, 0.2])
def test_barycenter_matches_oracle(floor):
    # NEXT-1 with the random-feature kernel (lambda > 0 as in the paper's runs,
    # PAPER.md:1061) against the fp64 oracle (Alg. 1, readings A20) after 1, 3
    # and 10 iterations and at the tol stop (same iteration count).  The
    # iteration amplifies FM_K errors (tests/test_oracle_integrator.py::
    # test_barycenter_conditioning_on_random_feature_kernels); the GPU keeps
    # v, w, d, mu in fp64 and FM_K's normwise error is ~1e-7
    # (tools/bary_trace.py, profiles/r02_bary_trace*.txt).
    from workloads import barycenter_inputs

    x, a, mus = barycenter_inputs(2000, floor=floor)
    plan = rfd.Plan(torch.from_numpy(x).cuda(), 0.03, 0.1, 256, 5)
    ref_plan = orf.Plan(x, 0.03, 0.1, 256, 5)
    for iters, tol in ((1, 0.0), (3, 0.0), (10, 0.0), (300, 1e-3)):
        got, its = _bary_gpu(plan, mus, a, [1 / 3] * 3, iters, tol=tol)
        ref, rits = ref_plan.barycenter(mus, a, [1 / 3] * 3, iters, tol=tol)
        err = relerr(got, ref)
        print("barycenter floor=%g iters=%d tol=%g: %d/%d iterations, err %.2e"
              % (floor, iters, tol, its, rits, err))
        assert its == rits
        assert err <= TOL
        assert np.isfinite(got).all() and (got >= 0).all()
        assert abs(float(a @ got) - 1.0) < 1e-5


@pytest.mark.parametrize("floor,iters,tol", [(0.0, 10, 0.0), (0.2, 10, 0.0), (0.0, 200, 1e-3)])
def test_barycenter_kernels_match_fp64_iteration(floor, iters, tol):
    # Past iteration 1 the random-feature barycenter is ill-conditioned in the
    # FM_K error (see the oracle conditioning test), so the elementwise GPU
    # steps are checked against the same iteration in fp64 driven by the same
    # GPU FM_K (bitwise-deterministic integrate on identically formed inputs):
    # 10 iterations and a tol stop, iterates, stop iteration and output.
    from workloads import barycenter_inputs

    x, a, mus = barycenter_inputs(2000, floor=floor)
    plan = rfd.Plan(torch.from_numpy(x).cuda(), 0.03, 0.1, 256, 5)
    got, its = _bary_gpu(plan, mus, a, [1 / 3] * 3, iters, tol=tol)
    ref, rits = _bary_hybrid(plan, mus, a, [1 / 3] * 3, iters, tol=tol)
    err = relerr(got, ref)
    print("barycenter floor=%g iters=%d tol=%g: %d/%d iterations, err vs fp64 iteration %.2e"
          % (floor, iters, tol, its, rits, err))
    assert its == rits
    assert err <= 1e-6
    assert np.isfinite(got).all() and (got >= 0).all()
    assert abs(float(a @ got) - 1.0) < 1e-5


def test_barycenter_errors():
    from workloads import barycenter_inputs

    x, a, mus = barycenter_inputs(2000)
    plan = rfd.Plan(torch.from_numpy(x).cuda(), 0.03, 0.1, 256, 5)
    mus_d = torch.from_numpy(mus.astype(np.float32)).cuda()
    a_d = torch.from_numpy(a.astype(np.float32)).cuda()
    for alpha in ([0.5, 0.5, 0.5], [1.0, 0.0, 0.0], [-1.0, 1.0, 1.0]):
        with pytest.raises(rfd.RFDError):
            plan.barycenter(mus_d, a_d, alpha, 3)
    with pytest.raises(ValueError):  # undersized inputs are refused by the binding
        plan.barycenter(mus_d[:, :100], a_d, [1 / 3] * 3, 3)
    with pytest.raises(ValueError):
        plan.barycenter(mus_d, a_d[:100], [1 / 3] * 3, 3)
    batched = rfd.Plan(torch.from_numpy(np.stack([x, x])).cuda(), 0.03, 0.1, 256, 5)
    with pytest.raises(rfd.RFDError):
        batched.barycenter(mus_d, a_d, [1 / 3] * 3, 3)


@pytest.mark.parametrize("n,m,seed,lam", [(1000, 40, 11, -0.8), (3001, 96, 14, -0.3),
                                          (2000, 128, 13, 0.05)])
def test_negative_nu_nonsymmetric_route(n, m, seed, lam):
    # eps = 0.2 puts some frequencies in a negative sinc lobe (nu < 0): the core
    # runs on lambda G D directly.  Where the oracle's exact result overflows
    # fp32 the library must refuse the plan with RFD_ERANGE instead.
    x = _sphere(n, seed)
    F = np.random.default_rng(seed).standard_normal((n, 3)).astype(np.float32)
    p = dict(name="nonsym n=%d m=%d" % (n, m), eps=0.2, lam=lam, m=m, seed=seed)
    ref = orf.Plan(x, p["eps"], p["lam"], p["m"], p["seed"])
    assert (ref.nu < 0).any()
    if not np.isfinite(ref.C).all() or np.abs(ref.C).max() > 1e30:
        with pytest.raises(rfd.RFDError) as ei:
            _run_single(x, F, p)
        assert ei.value.status == rfd.RFD_ERANGE
        return
    plan, out = _run_single(x, F, p)
    assert plan.info()["symmetric"] == 0
    _check_against_oracle(plan, out, x, F, p)


def test_single_point_closed_form():
    x = np.array([[0.3, -0.2, 0.9]], np.float32)
    F = np.array([[1.5, -2.0, 0.25, 4.0]], np.float32)
    plan, out = _run_single(x, F, dict(eps=0.1, lam=-0.6, m=16, seed=0))
    s = plan.export("nu").sum()
    np.testing.assert_allclose(out, math.exp(-0.6 * s) * F, rtol=2e-6)


def test_two_coincident_points_closed_form():
    x = np.array([[0.1, 0.2, 0.3], [0.1, 0.2, 0.3]], np.float32)
    F = np.array([[1.0, 2.0], [-3.0, 0.5]], np.float32)
    plan, out = _run_single(x, F, dict(eps=0.15, lam=-0.4, m=16, seed=1))
    s = plan.export("nu").sum()
    ref = F + 0.5 * math.expm1(2 * -0.4 * s) * np.ones((2, 2)) @ F
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-6)


def test_lambda_zero_is_exact_identity():
    x = _sphere(5000, 3)
    F = np.random.default_rng(0).standard_normal((5000, 3)).astype(np.float32)
    _, out = _run_single(x, F, dict(eps=0.1, lam=0.0, m=64, seed=2))
    np.testing.assert_array_equal(out, F)


def test_properties_determinism_inplace_linearity_symmetry_semigroup():
    p, x, F = make_config(2)
    xd = torch.from_numpy(x).cuda()
    Fd = torch.from_numpy(F).cuda()
    plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    a = plan.integrate(Fd)
    b = plan.integrate(Fd)
    assert torch.equal(a, b)  # bitwise deterministic
    plan2 = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    assert torch.equal(plan2.integrate(Fd), a)
    Fi = Fd.clone()
    plan.integrate(Fi, out=Fi)  # in place
    assert torch.equal(Fi, a)
    G2 = torch.randn_like(Fd)
    lin = plan.integrate(2 * Fd - G2)
    assert relerr((lin).cpu().numpy(), (2 * a - plan.integrate(G2)).cpu().numpy()) < 1e-5
    u = torch.randn(x.shape[0], 1, device="cuda")
    v = torch.randn(x.shape[0], 1, device="cuda")
    Ku, Kv = plan.integrate(u), plan.integrate(v)
    lhs, rhs = float((u * Kv).double().sum()), float((Ku * v).double().sum())
    assert abs(lhs - rhs) <= 1e-5 * abs(lhs)
    half = rfd.Plan(xd, p["eps"], p["lam"] / 2, p["m"], p["seed"])
    two = half.integrate(half.integrate(Fd))
    assert relerr(two.cpu().numpy(), a.cpu().numpy()) < 1e-4


@pytest.mark.parametrize("cfg", [1, 3, 4, 5])
def test_back_to_back_integrates_equal_synchronised(cfg):
    # Consecutive integrates overlap (programmatic dependent launch: pass 1's
    # setup runs during the previous pass 2, pass 2's during pass 1 /
    # core_apply).  Chains of in-place integrates, each output feeding the
    # next call, with no host synchronisation must equal the same chain run
    # with a device synchronisation after every call, bit for bit (fused a7
    # for cfgs 1 and 3; reduce_S + core_apply for cfgs 4 and 5).
    p, x, F = make_config(cfg)
    if cfg == 3:
        F = F[0]
    if cfg == 5:
        x, F = x[: 1 << 19], F[: 1 << 19]
    xd = torch.from_numpy(x).cuda()
    plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    F0 = torch.from_numpy(np.ascontiguousarray(F)).cuda()
    ref = F0.clone()
    outs_ref = []
    for _ in range(6):
        plan.integrate(ref, out=ref)
        torch.cuda.synchronize()
        outs_ref.append(ref.clone())
    # (separate buffers: no other kernel between one call's pass 2 and the
    # next call's pass 1)
    bufs = [F0] + [torch.empty_like(F0) for _ in range(6)]
    torch.cuda.synchronize()
    for k in range(6):
        plan.integrate(bufs[k], out=bufs[k + 1])
    torch.cuda.synchronize()
    for a, b in zip(bufs[1:], outs_ref):
        assert torch.equal(a, b)
    # the same chain in place, back to back
    cur = F0.clone()
    torch.cuda.synchronize()
    for _ in range(6):
        plan.integrate(cur, out=cur)
    torch.cuda.synchronize()
    assert torch.equal(cur, outs_ref[-1])


def test_host_buffers_match_device():
    p, x, F = make_config(4)
    plan = rfd.Plan(x, p["eps"], p["lam"], p["m"], p["seed"])  # host points
    Fh = torch.from_numpy(F).pin_memory()
    oh = torch.empty_like(Fh).pin_memory()
    plan.integrate_host(Fh, oh)
    torch.cuda.synchronize()
    od = plan.integrate(Fh.cuda()).cpu()
    assert torch.equal(oh, od)  # d <= 4: the same one-launch path


def test_overflow_reports_erange():
    p, x, F = make_config(2)
    with pytest.raises(rfd.RFDError) as ei:
        rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], 200.0, p["m"], p["seed"])
    assert ei.value.status == rfd.RFD_ERANGE
    # rfd_gfi checks the core's overflow flag only after the inference is
    # enqueued (plan.cu core_finish): the error still surfaces, on the narrow
    # path, the tensor-core path and the spread-grid path (its early powers),
    # and the next call on the same thread is unaffected
    for cfg, kw, d in ((2, {}, 1), (2, {}, 8), (5, {"n": 262144}, 16)):
        p, x, F = make_config(cfg, **kw)
        xd = torch.from_numpy(x).cuda()
        Fd = torch.from_numpy(np.ascontiguousarray(F.reshape(x.shape[0], -1)[:, :1])).cuda()
        Fd = Fd.repeat(1, d).contiguous()
        with pytest.raises(rfd.RFDError) as ei:
            rfd.gfi(xd, p["eps"], 200.0, p["m"], p["seed"], Fd)
        assert ei.value.status == rfd.RFD_ERANGE
        out = rfd.gfi(xd, p["eps"], p["lam"], p["m"], p["seed"], Fd)
        ref = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"]).integrate(Fd)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)


def test_cuda_graph_capture_of_reuse_loop():
    p, x, V = make_config(3)
    xd = torch.from_numpy(x).cuda()
    plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
    Vd = torch.from_numpy(V[:10]).cuda()
    eager = torch.stack([plan.integrate(Vd[t]) for t in range(10)])
    outs = torch.empty_like(Vd)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        plan.integrate(Vd[0], out=outs[0])  # workspace sized before capture
        with torch.cuda.graph(g, stream=s):
            for t in range(10):
                plan.integrate(Vd[t], out=outs[t], stream=s)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(outs, eager)


def test_launch_counter_and_profiler():
    p, x, F = make_config(1)
    c0 = rfd.launch_count()
    plan = rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
    rfd.profile_enable(True)
    plan.integrate(torch.from_numpy(F).cuda())
    prof = rfd.profile_read()
    rfd.profile_enable(False)
    assert rfd.launch_count() > c0
    # d = 3 <= 4: one cooperative launch does the whole inference
    assert set(prof) == {"rfd_integrate_small"}
    assert all(v[1] > 0 for v in prof.values())
    # r = 32, d = 8: tensor-core passes with a7 fused in pass 2
    rfd.profile_enable(True)
    plan.integrate(torch.from_numpy(np.ones((x.shape[0], 8), np.float32)).cuda())
    prof8 = rfd.profile_read()
    rfd.profile_enable(False)
    assert set(prof8) == {"rfd_pass1_tc", "rfd_pass2_tc"}
    # r = 256, d = 8: the separate a7 kernels
    x4 = _sphere(4000, 3)
    plan4 = rfd.Plan(torch.from_numpy(x4).cuda(), 0.05, -0.8, 128, 3)
    rfd.profile_enable(True)
    plan4.integrate(torch.from_numpy(np.ones((4000, 8), np.float32)).cuda())
    prof4 = rfd.profile_read()
    rfd.profile_enable(False)
    assert {"rfd_reduce_S", "rfd_core_apply", "rfd_pass1_tc", "rfd_pass2_tc"} <= set(prof4)


@pytest.mark.parametrize("cfg,n,shift", [(4, None, 0.0), (5, 262144, 0.0), (5, 262144, 1000.0),
                                         (4, None, 100.0)])
def test_gram_spread_grid_parity(cfg, n, shift, monkeypatch):
    # a4 through the spread grid (k_nufft.cu) against the oracle's direct sum
    # and against the direct tensor-core Gram; bitwise deterministic (integer
    # spreading) and exactly symmetric.  RFD_GRAM_SPREAD=2 forces the grid,
    # =0 the direct path (the default picks the grid when it has <= n/8 nodes).
    p, x, F = make_config(cfg, **({"n": n} if n else {}))
    x = (x.astype(np.float64) + shift * np.array([1.0, -0.7, 0.4])).astype(np.float32)
    p = dict(p, name="cfg%d n %d shift %g" % (cfg, x.shape[0], shift))
    ref = orf.Plan(x, p["eps"], p["lam"], p["m"], p["seed"])
    res = ref.apply(F.astype(np.float64))
    F2 = F.reshape(F.shape[0], -1).astype(np.float64)
    Gs = {}
    for mode in ("0", "2"):
        monkeypatch.setenv("RFD_GRAM_SPREAD", mode)
        plan, out = _run_single(x, F, p)
        nodes = plan.info()["gram_nodes"]
        assert (nodes > 0) == (mode == "2"), nodes
        G = plan.export("gram")
        Gs[mode] = G
        o2 = out.reshape(out.shape[0], -1)
        errs = dict(G=relerr(G, ref.G), C=relerr(plan.export("core"), ref.C),
                    out=relerr(o2, res["out"]), delta=relerr(o2 - F2, res["out"] - F2))
        print(p["name"], "mode", mode, "nodes", nodes, {k: "%.2e" % v for k, v in errs.items()})
        assert errs["G"] <= 2e-5 and max(errs.values()) <= TOL, errs
        if mode == "2":
            G2 = _run_single(x, F, p)[0].export("gram")
            np.testing.assert_array_equal(G, G2)
            assert relerr(G, G.T) <= 1e-15  # the export's rotation back rounds
    assert relerr(Gs["2"], Gs["0"]) <= 2e-5


@pytest.mark.parametrize("cfg,n,spread", [(1, None, "1"), (2, None, "1"), (5, 262144, "2"),
                                          (5, 262144, "0")])
def test_gfi_one_shot_equals_plan_and_integrate(cfg, n, spread, monkeypatch):
    # rfd_gfi runs pass 1 on a second stream beside the plan's core: same
    # kernels, so bitwise the two-call result; the returned plan is reusable
    monkeypatch.setenv("RFD_GRAM_SPREAD", spread)
    p, x, F = make_config(cfg, **({"n": n} if n else {}))
    xd, Fd = torch.from_numpy(x).cuda(), torch.from_numpy(np.ascontiguousarray(F)).cuda()
    ref = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"]).integrate(Fd)
    out = rfd.gfi(xd, p["eps"], p["lam"], p["m"], p["seed"], Fd)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    out2, plan = rfd.gfi(x, p["eps"], p["lam"], p["m"], p["seed"], Fd, keep_plan=True)  # host points
    assert torch.equal(out2, ref)
    assert torch.equal(plan.integrate(Fd), ref)
    with pytest.raises(rfd.RFDError):
        rfd.gfi(xd, p["eps"], p["lam"], p["m"], p["seed"], torch.from_numpy(np.ascontiguousarray(F)),
                torch.empty_like(Fd))


@pytest.mark.parametrize("mode", ["0", "2"])
@pytest.mark.parametrize("shape", ["point", "line", "plane"])
def test_gram_spread_grid_degenerate_extents(shape, mode, monkeypatch):
    # zero extent on 3, 2 or 1 axes: the grid shrinks to the kernel's width on
    # those axes (L = ceil(alpha / h) + 1); forced through the spread path
    monkeypatch.setenv("RFD_GRAM_SPREAD", mode)
    rng = np.random.default_rng(11)
    n = 4096
    x = np.zeros((n, 3))
    if shape != "point":
        x[:, 0] = rng.uniform(-0.5, 0.5, n)
    if shape == "plane":
        x[:, 1] = rng.uniform(-0.3, 0.3, n)
    x = (x + np.array([0.25, -1.0, 3.0])).astype(np.float32)
    F = rng.standard_normal((n, 8)).astype(np.float32)
    p = dict(name="spread " + shape, eps=0.05, lam=-0.4, m=128, seed=6)
    plan, out = _run_single(x, F, p)
    assert (plan.info()["gram_nodes"] > 0) == (mode == "2")
    _check_against_oracle(plan, out, x, F, p)


def test_gram_spread_grid_cell_beyond_fold(monkeypatch):
    # 9,000 coincident points (one grid cell: more than the tensor-core
    # spread's 8192 points per exact class-sum fold, so the fold carries its
    # remainder, k_nufft.cu) among 13,000 spread ones; parity and bitwise
    # determinism as everywhere else.  (A heavier coincident mass makes the
    # core ill-conditioned on either Gram path: 20,000 + 2,000 points give
    # Delta 2.8e-5 direct, 6.0e-5 spread; tools/fold_cmp.py.)
    monkeypatch.setenv("RFD_GRAM_SPREAD", "2")
    rng = np.random.default_rng(5)
    n = 22000
    x = np.empty((n, 3))
    x[:9000] = np.array([0.1, 0.2, -0.3])
    x[9000:] = rng.uniform(-0.5, 0.5, (13000, 3))
    x = x.astype(np.float32)
    F = rng.standard_normal((n, 4)).astype(np.float32)
    p = dict(name="spread one cell", eps=0.05, lam=-0.4, m=128, seed=2)
    plan, out = _run_single(x, F, p)
    assert plan.info()["gram_nodes"] > 0
    np.testing.assert_array_equal(plan.export("gram"), _run_single(x, F, p)[0].export("gram"))
    _check_against_oracle(plan, out, x, F, p)


@pytest.mark.parametrize("offset", [0, 1, 2, 3])
def test_bounding_box_misaligned_points_and_extremes(offset, monkeypatch):
    # The bounding box (k_freq.cu bbox_kernel) reads whole points as float4
    # triples from the first 16-byte boundary on, the head and the ragged
    # tail by scalar loads: the extreme points sit exactly there (indices 0-2
    # and the last two), the cloud starts `offset` floats past a 16-byte
    # boundary, and n is odd.  The box sizes a4's spread grid, so a missed
    # point would change the node count (and put the point off the grid);
    # a view and a copy of the same points give bitwise the same plan.
    monkeypatch.setenv("RFD_GRAM_SPREAD", "2")
    rng = np.random.default_rng(17)
    n = 6001
    x = rng.uniform(-0.2, 0.2, (n, 3))
    x[0] = [0.9, 0.0, 0.0]
    x[1] = [0.0, -0.8, 0.0]
    x[2] = [0.0, 0.0, 0.7]
    x[n - 2] = [-0.6, 0.0, 0.0]
    x[n - 1] = [0.0, 0.5, -0.9]
    x = x.astype(np.float32)
    buf = torch.zeros(3 * n + 8, dtype=torch.float32, device="cuda")
    buf[offset:offset + 3 * n] = torch.from_numpy(x.reshape(-1)).cuda()
    view = buf[offset:offset + 3 * n].view(n, 3)
    assert (view.data_ptr() % 16) == 4 * offset
    p = dict(name="bbox offset %d" % offset, eps=0.05, lam=-0.4, m=128, seed=4)
    F = rng.standard_normal((n, 5)).astype(np.float32)
    plan_v = rfd.Plan(view, p["eps"], p["lam"], p["m"], p["seed"])
    plan_c, out_c = _run_single(x, F, p)
    assert plan_v.info()["gram_nodes"] == plan_c.info()["gram_nodes"] > 0
    np.testing.assert_array_equal(plan_v.export("gram"), plan_c.export("gram"))
    out_v = plan_v.integrate(torch.from_numpy(F).cuda()).cpu().numpy()
    np.testing.assert_array_equal(out_v, out_c)
    _check_against_oracle(plan_c, out_c, x, F, p)


def test_gram_spread_grid_scan_variants_agree(monkeypatch):
    # the cell-start scan: one CTA for grids of <= 2^18 cells, two tiled
    # kernels above (forced here: RFD_NUFFT_SCAN_TILES=1); the exact integer
    # spreading makes G bitwise independent of the point order in a cell
    monkeypatch.setenv("RFD_GRAM_SPREAD", "2")
    p, x, F = make_config(4)
    plan1, out1 = _run_single(x, F, p)
    monkeypatch.setenv("RFD_NUFFT_SCAN_TILES", "1")
    plan2, out2 = _run_single(x, F, p)
    assert plan1.info()["gram_nodes"] == plan2.info()["gram_nodes"] > 4096
    np.testing.assert_array_equal(plan1.export("gram"), plan2.export("gram"))
    np.testing.assert_array_equal(out1, out2)


def test_gram_spread_grid_declines_large_extent(monkeypatch):
    # cfg 4's sheet scaled x 200 would need > 2^11 nodes per axis: even
    # forced, the plan takes the direct Gram
    monkeypatch.setenv("RFD_GRAM_SPREAD", "2")
    p, x, F = make_config(4)
    plan, _ = _run_single((x * 200.0).astype(np.float32), F, p)
    assert plan.info()["gram_nodes"] == 0


@pytest.mark.parametrize("d", [1, 2, 3, 4])
def test_narrow_field_paths_agree(d, monkeypatch):
    # the d <= 4 one-launch SIMT path (forced: RFD_NARROW=2) and the
    # tensor-core passes (the same columns inside a d = 8 field) against each
    # other and the oracle
    monkeypatch.setenv("RFD_NARROW", "2")
    p, x, F = make_config(4)
    rng = np.random.default_rng(d)
    F8 = rng.standard_normal((x.shape[0], 8)).astype(np.float32)
    plan = rfd.Plan(torch.from_numpy(x).cuda(), p["eps"], p["lam"], p["m"], p["seed"])
    o8 = plan.integrate(torch.from_numpy(F8).cuda()).cpu().numpy()
    od = plan.integrate(torch.from_numpy(np.ascontiguousarray(F8[:, :d])).cuda()).cpu().numpy()
    ref = orf.Plan(x, p["eps"], p["lam"], p["m"], p["seed"]).apply(F8[:, :d].astype(np.float64))["out"]
    F64 = F8[:, :d].astype(np.float64)
    for got in (od, o8[:, :d]):
        assert relerr(got, ref) <= TOL
        assert relerr(got - F64, ref - F64) <= TOL
    assert relerr(od - F64, o8[:, :d] - F64) <= 2e-5


@pytest.mark.parametrize("lam,cases", [(0.1, ((3, 0.0), (10, 0.0), (300, 1e-3))),
                                       (0.5, ((3, 0.0), (10, 0.0)))])
def test_barycenter_fused_matches_oracle_and_unfused(lam, cases, monkeypatch):
    # NEXT-1 fused (k_bary_fused.cu: m <= 32, k <= 4, n <= 148 x 512 -- the
    # paper's barycenter regime, m = 30): the whole Alg. 1 loop
    # in one launch with the feature rows cached on chip.  Iteration 1 against
    # the fp64 oracle; later iterations amplify the FM_K error (at m = 30 both
    # GPU paths sit ~2e-4 from the oracle after 2-10 iterations at lambda = 0.1,
    # tools/bary_fused_check.py), so there the fused loop is checked against
    # the unfused one (same FM_K arithmetic class, gated against the oracle at
    # 10 iterations by test_barycenter_matches_oracle): <= 1e-5, same stop.
    from workloads import barycenter_inputs

    x, a, mus = barycenter_inputs(3000)
    plan = rfd.Plan(torch.from_numpy(x).cuda(), 0.03, lam, 30, 5)
    ref, _ = orf.Plan(x, 0.03, lam, 30, 5).barycenter(mus, a, [1 / 3] * 3, 1)
    rfd.profile_enable(True)
    rfd.profile_read()
    got, its = _bary_gpu(plan, mus, a, [1 / 3] * 3, 1)
    prof = rfd.profile_read()
    rfd.profile_enable(False)
    assert set(prof) == {"rfd_bary_fused"}  # one launch per call, nothing else
    err = relerr(got, ref)
    print("fused barycenter lam=%g iteration 1: err %.2e" % (lam, err))
    assert its == 1 and err <= TOL
    # (lambda = 0.5's tol stop runs ~20 iterations on inputs where the oracle
    # itself moves 7.6e-4 under 1e-7 FM_K noise: not a meaningful 1e-5 check)
    for iters, tol in cases:
        f, fits = _bary_gpu(plan, mus, a, [1 / 3] * 3, iters, tol=tol)
        monkeypatch.setenv("RFD_BARY_FUSED", "0")
        u, uits = _bary_gpu(plan, mus, a, [1 / 3] * 3, iters, tol=tol)
        monkeypatch.delenv("RFD_BARY_FUSED")
        e = relerr(f, u)
        print("fused vs unfused lam=%g iters=%d tol=%g: %d/%d iterations, %.2e" % (lam, iters, tol, fits, uits, e))
        assert fits == uits
        assert e <= 1e-5
        assert abs(float(a @ f) - 1.0) < 1e-5


def test_barycenter_fused_closed_form_and_fallback():
    from workloads import barycenter_inputs

    x, a, mus = barycenter_inputs(3000, floor=0.05)
    # identity kernel (lambda = 0): the geometric mean at every iteration
    plan0 = rfd.Plan(torch.from_numpy(x).cuda(), 0.03, 0.0, 16, 5)
    m32 = mus.astype(np.float32).astype(np.float64)
    a32 = a.astype(np.float32).astype(np.float64)
    geo = np.prod(m32 ** (1 / 3), axis=0)
    geo /= a32 @ geo
    rfd.profile_enable(True)
    rfd.profile_read()
    got, its = _bary_gpu(plan0, mus, a, [1 / 3] * 3, 5)
    assert set(rfd.profile_read()) == {"rfd_bary_fused"}
    assert its == 5 and relerr(got, geo) <= 1e-6
    # m > 32: the unfused path
    plan64 = rfd.Plan(torch.from_numpy(x).cuda(), 0.03, 0.0, 64, 5)
    got, its = _bary_gpu(plan64, mus, a, [1 / 3] * 3, 2)
    assert "rfd_bary_fused" not in rfd.profile_read()
    rfd.profile_enable(False)
    assert relerr(got, geo) <= 1e-6
