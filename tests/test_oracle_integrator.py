"""Pins for the whole oracle integrator and the dense diagnostic (no GPU).

The closed form must equal exp(lambda Phi D Phi^T) F exactly (up to
rounding) -- it is an identity of the low-rank matrix,
not an approximation -- so it is checked against a dense matrix exponential
computed by a different algorithm (symmetric eigendecomposition / scipy
expm), plus closed forms, invariants and limits.
"""

import math

import numpy as np
import pytest
import scipy.linalg

from oracle import dense, rfd

C_R = rfd.l1_ball_mass()


def _lowrank_dense(plan):
    """W~ = Phi D Phi^T as an explicit N x N matrix (tiny N only)."""
    P = rfd.features(plan.X, plan.omega)
    d = np.concatenate([plan.nu, plan.nu])
    return P @ (d[:, None] * P.T)


def _cloud(n, seed=0):
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, 3))
    return (g / np.linalg.norm(g, axis=1, keepdims=True)).astype(np.float32), rng


@pytest.mark.parametrize("n,m,eps,lam", [(300, 8, 0.3, -0.7), (1000, 16, 0.15, -0.5),
                                         (600, 64, 0.2, -1.5), (400, 32, 0.25, 0.4)])
def test_identity_against_dense_expm(n, m, eps, lam):
    X, rng = _cloud(n, seed=n)
    F = rng.standard_normal((n, 3))
    plan = rfd.Plan(X, eps, lam, m, seed=7, c_r=C_R)
    out = plan.apply(F)["out"]
    ref = dense.symmetric_expm_apply(_lowrank_dense(plan), lam, F)
    assert np.abs(out - ref).max() <= 1e-10 * np.abs(ref).max()


def test_identity_against_scipy_expm_small():
    X, rng = _cloud(120, seed=3)
    F = rng.standard_normal((120, 2))
    plan = rfd.Plan(X, 0.3, -0.8, 12, seed=2, c_r=C_R)
    ref = scipy.linalg.expm(-0.8 * _lowrank_dense(plan)) @ F
    out = plan.apply(F)["out"]
    assert np.abs(out - ref).max() <= 1e-11 * np.abs(ref).max()


def test_single_point_closed_form():
    X = np.array([[0.3, -0.2, 0.9]], np.float32)
    F = np.array([[1.5, -2.0, 0.25]])
    plan = rfd.Plan(X, 0.1, -0.6, 16, seed=0, c_r=C_R)
    out = plan.apply(F)["out"]
    np.testing.assert_allclose(out, math.exp(-0.6 * plan.nu.sum()) * F, rtol=1e-13)


def test_two_coincident_points_closed_form():
    X = np.array([[0.1, 0.2, 0.3], [0.1, 0.2, 0.3]], np.float32)
    F = np.array([[1.0, 2.0], [-3.0, 0.5]])
    lam = -0.4
    plan = rfd.Plan(X, 0.15, lam, 16, seed=1, c_r=C_R)
    s = plan.nu.sum()
    ref = F + 0.5 * math.expm1(2 * lam * s) * np.ones((2, 2)) @ F
    np.testing.assert_allclose(plan.apply(F)["out"], ref, rtol=1e-13, atol=1e-14)


def test_first_order_in_lambda():
    X, rng = _cloud(200, seed=5)
    F = rng.standard_normal((200, 3))
    lam = 1e-6
    plan = rfd.Plan(X, 0.2, lam, 16, seed=4, c_r=C_R)
    first = _lowrank_dense(plan) @ F
    got = (plan.apply(F)["out"] - F) / lam
    assert np.abs(got - first).max() <= 1e-4 * np.abs(first).max()


def test_lambda_zero_identity():
    X, rng = _cloud(50, seed=6)
    F = rng.standard_normal((50, 3))
    plan = rfd.Plan(X, 0.2, 0.0, 8, seed=4, c_r=C_R)
    np.testing.assert_array_equal(plan.apply(F)["out"], F)


def test_semigroup_symmetry_linearity_permutation():
    X, rng = _cloud(300, seed=8)
    F = rng.standard_normal((300, 2))
    lam = -0.7
    full = rfd.Plan(X, 0.3, lam, 8, seed=3, c_r=C_R)
    half = rfd.Plan(X, 0.3, lam / 2, 8, seed=3, c_r=C_R)
    a = full.apply(F)["out"]
    b = half.apply(half.apply(F)["out"])["out"]
    assert np.abs(a - b).max() <= 1e-12 * np.abs(a).max()
    u = rng.standard_normal(300)
    v = rng.standard_normal(300)
    Ku = full.apply(u)["out"][:, 0]
    Kv = full.apply(v)["out"][:, 0]
    assert abs(u @ Kv - Ku @ v) <= 1e-12 * abs(u @ Kv)
    G2 = rng.standard_normal((300, 2))
    np.testing.assert_allclose(full.apply(2 * F - G2)["out"], 2 * a - full.apply(G2)["out"],
                               atol=1e-11)
    perm = rng.permutation(300)
    pplan = rfd.Plan(X[perm], 0.3, lam, 8, seed=3, c_r=C_R)
    np.testing.assert_allclose(pplan.apply(F[perm])["out"], a[perm], atol=1e-11)


def test_reparam_keeps_gram_and_matches_dense():
    # NEXT-4: G depends on the points and omega only; after a
    # re-parameterisation the integrator must equal the dense exponential of
    # the NEW low-rank W~ (an independent route) and a fresh plan.
    X, rng = _cloud(400, seed=12)
    F = rng.standard_normal((400, 2))
    plan = rfd.Plan(X, 0.3, -0.7, 16, seed=6, c_r=C_R)
    G0 = plan.G.copy()
    plan.reparam(0.18, -1.3)
    np.testing.assert_array_equal(plan.G, G0)
    fresh = rfd.Plan(X, 0.18, -1.3, 16, seed=6, c_r=C_R)
    np.testing.assert_array_equal(plan.nu, fresh.nu)
    np.testing.assert_array_equal(plan.C, fresh.C)
    out = plan.apply(F)["out"]
    ref = dense.symmetric_expm_apply(_lowrank_dense(plan), -1.3, F)
    assert np.abs(out - ref).max() <= 1e-10 * np.abs(ref).max()


@pytest.mark.parametrize("n,m,lam", [(150, 6, -0.8), (300, 16, -0.3), (10, 8, -0.6),
                                     (40, 24, 0.3)])
def test_spectrum_against_dense_eigendecomposition(n, m, lam):
    # NEXT-3: the low-rank route equals the k smallest
    # eigenvalues of the dense N x N exp(lam W~) (brute force), including
    # N < 2m (reading A19) and lambda > 0.
    X, rng = _cloud(n, seed=n + m)
    plan = rfd.Plan(X, 0.3, lam, m, seed=9, c_r=C_R)
    W = _lowrank_dense(plan)
    ref = np.sort(np.exp(lam * np.linalg.eigvalsh(W)))
    for k in (1, min(n, 5), n):
        np.testing.assert_allclose(plan.spectrum(k), ref[:k], rtol=0, atol=1e-9 * ref.max())


def test_spectrum_special_cases():
    # lambda = 0: K = I; rank-1 A = B = e1, lambda > 0, k = 2,
    # N >= 3 gives [1, 1] -- here through G = e1 e1^T, nu = 1.
    X, _ = _cloud(50, seed=1)
    plan = rfd.Plan(X, 0.3, 0.0, 8, seed=2, c_r=C_R)
    np.testing.assert_array_equal(plan.spectrum(7), np.ones(7))
    G = np.zeros((2, 2))
    G[0, 0] = 1.0
    np.testing.assert_array_equal(rfd.spectrum(G, np.array([1.0]), 0.7, 3, 2), [1.0, 1.0])
    np.testing.assert_allclose(rfd.spectrum(G, np.array([1.0]), 0.7, 3, 3)[-1], math.exp(0.7))


def _bumps(X, centers, sigma):
    X = np.asarray(X, np.float64)
    return np.stack([np.exp(-((X - np.asarray(c, np.float64)) ** 2).sum(1) / (2 * sigma ** 2))
                     for c in centers])


def test_barycenter_identity_kernel_fixed_point():
    # FM = identity (lambda = 0), a uniform, k = 1 -> mu = mu^1
    # after one iteration (the iteration is w = mu1 / v, d = v w = mu1, mu = d).
    X, rng = _cloud(200, seed=4)
    a = np.full(200, 1.0 / 200)
    mu1 = _bumps(X, [X[0]], 0.5)
    mu1 /= a @ mu1[0]
    plan = rfd.Plan(X, 0.3, 0.0, 8, seed=1, c_r=C_R)
    mu, it = plan.barycenter(mu1, a, [1.0], 1)
    np.testing.assert_allclose(mu, mu1[0], rtol=1e-12)


def test_barycenter_against_dense_kernel_and_symmetry():
    # Alg. 1 with FM = the RFD closed form equals Alg. 1 with FM = the dense
    # exp(lam W~) (independent route); identical inputs give d^1 = d^2, i.e.
    # the same barycenter as the single input with alpha = 1.
    X, rng = _cloud(300, seed=6)
    a = np.full(300, 1.0 / 300)
    mus = _bumps(X, [X[0], X[100], X[200]], 0.6)
    mus /= (mus @ a)[:, None]
    lam = 0.5
    plan = rfd.Plan(X, 0.3, lam, 12, seed=3, c_r=C_R)
    W = _lowrank_dense(plan)
    dense = lambda Y: dense_apply(W, lam, Y)
    alpha = [1 / 3, 1 / 3, 1 / 3]
    mu_rfd, _ = plan.barycenter(mus, a, alpha, 8)
    mu_dense, _ = rfd.barycenter(dense, mus, a, alpha, 8)
    np.testing.assert_allclose(mu_rfd, mu_dense, rtol=1e-8)
    two, _ = plan.barycenter(np.stack([mus[1], mus[1]]), a, [0.5, 0.5], 8)
    one, _ = plan.barycenter(mus[1:2], a, [1.0], 8)
    np.testing.assert_allclose(two, one, rtol=1e-10)
    assert abs(a @ mu_rfd - 1.0) < 1e-12


def dense_apply(W, lam, Y):
    return dense.symmetric_expm_apply(W, lam, Y)


def test_rows_subset_matches_full():
    X, rng = _cloud(500, seed=9)
    F = rng.standard_normal((500, 4))
    plan = rfd.Plan(X, 0.2, -1.0, 16, seed=5, c_r=C_R)
    full = plan.apply(F)["out"]
    rows = np.array([0, 17, 499, 250])
    np.testing.assert_allclose(plan.apply(F, rows=rows)["out"], full[rows], rtol=1e-14, atol=1e-14)


def _median_mse(m, norm, seeds=20):
    X, _ = _cloud(400, seed=11)
    eps = 0.15
    truth = dense.epsilon_graph(X, eps, norm)
    P_cache = []
    mses = []
    for s in range(seeds):
        om, _ = rfd.frequencies(1000 + s, m)
        nu = rfd.importance_weights(om, eps, C_R)
        P = rfd.features(X, om)
        W = P @ (np.concatenate([nu, nu])[:, None] * P.T)
        mses.append(np.mean((W - truth) ** 2))
    del P_cache
    return float(np.median(mses))


def test_adjacency_error_falls_with_m_and_is_cube_graph():
    # Approximation quality vs the exact graph: parity unpinned; trend only
    # (Lemma 2.7's 1/m variance term; A2, A9).
    inf16, inf256 = _median_mse(16, "inf"), _median_mse(256, "inf")
    assert inf256 < 0.5 * inf16
    assert inf16 < _median_mse(16, 1)


def test_barycenter_geometric_mean_pin():
    # Alg. 1 step 3 is a weighted GEOMETRIC mean of the d^i.
    # With FM = identity, d^i = v^i (a w^i) = v^i a mu^i / (a v^i) = mu^i for
    # any v and a, so every iteration gives mu = prod_i (mu^i)^alpha_i, then
    # <a, mu> = 1.  Two distinct inputs and alpha = (1/4, 3/4) separate this
    # from an arithmetic mean (or from swapped weights) by O(1).
    X, rng = _cloud(300, seed=12)
    a = rng.uniform(0.5, 1.5, 300)
    a /= a.sum()
    mus = _bumps(X, [X[3], X[200]], 0.4) + 0.05
    mus /= (mus @ a)[:, None]
    alpha = [0.25, 0.75]
    geo = mus[0] ** 0.25 * mus[1] ** 0.75
    geo /= a @ geo
    ari = 0.25 * mus[0] + 0.75 * mus[1]
    swp = mus[0] ** 0.75 * mus[1] ** 0.25
    swp /= a @ swp
    for iters in (1, 4):
        mu, it = rfd.barycenter(lambda Y: Y, mus, a, alpha, iters)
        assert it == iters
        np.testing.assert_allclose(mu, geo, rtol=1e-12)
        assert np.abs(mu - ari).max() > 0.1 * np.abs(geo).max()
        assert np.abs(mu - swp).max() > 0.1 * np.abs(geo).max()
    # the fixed point is reached at iteration 1: ||mu_2 - mu_1||_1 = 0 < tol
    _, it = rfd.barycenter(lambda Y: Y, mus, a, alpha, 50, tol=1e-12)
    assert it == 2


def test_barycenter_clamp_and_error():
    # denominators clamped at 1e-30; a non-finite iterate is an
    # error naming the iteration.  A kernel mapping everything to 0 makes both
    # denominators clamp: w = mu / 1e-30, d = max(v * 0, 1e-30) = 1e-30, so
    # mu = 1e-30 everywhere and v is unchanged (mu / d = 1).
    n = 50
    a = np.full(n, 1.0 / n)
    mus = np.ones((2, n))
    mu, it = rfd.barycenter(lambda Y: 0.0 * Y, mus, a, [0.5, 0.5], 3)
    np.testing.assert_allclose(mu, np.ones(n), rtol=1e-12)  # normalised 1e-30 * ones
    assert rfd.BARY_CLAMP == 1e-30
    with pytest.raises(FloatingPointError, match="iteration 1"):
        rfd.barycenter(lambda Y: np.full_like(Y, np.inf), mus, a, [0.5, 0.5], 3)


def test_barycenter_conditioning_on_random_feature_kernels():
    # DESIGN.md A20 (numerics): Alg. 1 divides by FM_K outputs, so it amplifies
    # FM_K errors; how much is heavy-tailed (an entry near the clamp can flip).
    # On the GPU test's inputs (workloads.barycenter_inputs), with every FM_K
    # output perturbed uniformly by eta of its column max:
    #   * iteration 1 on the floored inputs moves linearly, ~2.5 eta;
    #   * 10 iterations stay within 2e-5 at eta = 1e-7 (GPU FM_K errors are
    #     1e-8 .. 6e-7, tools/bary_trace.py), but eta = 1e-6 can move the
    #     floored inputs' result by O(1).
    # So a 1e-4 gate after 10 iterations holds only for an FM_K accurate to
    # ~1e-7 -- fp32 iterates (the round-1 design) could not meet it.
    from workloads import barycenter_inputs

    x, a, mus = barycenter_inputs(2000)
    _, _, mus_f = barycenter_inputs(2000, floor=0.2)
    plan = rfd.Plan(x, 0.03, 0.1, 256, seed=5, c_r=C_R)

    def moved(m, iters, eta, reps=3):
        ref, _ = plan.barycenter(m, a, [1 / 3] * 3, iters)
        g = np.random.default_rng(1)

        def noisy(Y):
            o = plan.apply(Y)["out"]
            return o + eta * np.abs(o).max(axis=0)[None, :] * g.uniform(-1, 1, o.shape)
        return [np.abs(rfd.barycenter(noisy, m, a, [1 / 3] * 3, iters)[0] - ref).max()
                / np.abs(ref).max() for _ in range(reps)]

    well = moved(mus_f, 1, 1e-5)
    assert max(well) < 5e-5 and min(well) > 1e-6
    assert max(moved(mus, 10, 1e-7)) < 2e-5
    assert max(moved(mus_f, 10, 1e-6)) > 0.5
