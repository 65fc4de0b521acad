"""Pins for the step functions of oracle/rfd.py (a1..a6), no GPU.

Each check is against something other than the oracle's own formula: a value
printed in SPEC.md, a closed form, a numerical quadrature, a Monte-Carlo
estimate, brute force, or an invariant the mathematics fixes.
"""

import math

import numpy as np
import pytest
import scipy.integrate
import scipy.linalg
import scipy.stats

import json
import os

from oracle import rfd

C_R = rfd.l1_ball_mass()
PINS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))


# ---------------------------------------------------------------- a2: tau
def test_tau_at_zero_is_box_volume():
    for eps in (0.01, 0.15, 0.5):
        assert rfd.tau(np.zeros(3), eps) == pytest.approx((2 * eps) ** 3, rel=1e-15)


def test_tau_spec_negative_lobe_value():
    # eps = 1, omega = (0.6, 0, 0) -> approx -1.247.
    pin = PINS["tau_negative_lobe"]
    assert rfd.tau(np.array(pin["omega"]), pin["eps"]) == pytest.approx(pin["value"], abs=pin["abs_tol"])


@pytest.mark.parametrize("eps,w", [(0.15, 0.6), (0.01, 3.3), (0.08, -1.7), (1.0, 0.25)])
def test_tau_factor_is_fourier_integral_of_interval(eps, w):
    # int_{-eps}^{eps} exp(-2 pi i w z) dz = int cos(2 pi w z) dz  (PAPER.md:310
    # convention), by adaptive quadrature.
    q, _ = scipy.integrate.quad(lambda z: math.cos(2 * math.pi * w * z), -eps, eps,
                                epsabs=1e-14, epsrel=1e-13)
    assert rfd.tau(np.array([w, 0.0, 0.0]), eps) / (2 * eps) ** 2 == pytest.approx(q, rel=1e-10, abs=1e-14)


def test_tau_is_separable_product():
    w = np.array([0.3, -1.1, 2.2])
    eps = 0.2
    parts = [rfd.tau(np.array([c, 0.0, 0.0]), eps) / (2 * eps) ** 2 for c in w]
    assert rfd.tau(w, eps) == pytest.approx(np.prod(parts), rel=1e-13)


def test_inverse_transform_of_1d_factor_is_interval_indicator():
    # int cos(2 pi w z) s(w) dw = 1[|z| <= eps] (Dirichlet integral), truncated
    # at |w| <= W: error O(1 / (W |z +- eps|)).
    eps, W = 0.15, 400.0
    s = lambda w: rfd.tau(np.array([w, 0.0, 0.0]), eps) / (2 * eps) ** 2
    for z, want in ((0.05, 1.0), (0.0, 1.0), (0.3, 0.0), (0.5, 0.0)):
        val, _ = scipy.integrate.quad(lambda w: math.cos(2 * math.pi * w * z) * s(w),
                                      -W, W, limit=20000, epsabs=1e-10)
        assert val == pytest.approx(want, abs=5e-3)


# ---------------------------------------------------------------- a2: C_R
def test_c_r_monte_carlo_small_radius():
    rng = np.random.default_rng(7)
    z = rng.standard_normal((2_000_000, 3))
    for R in (1.0, 2.0):
        p = np.mean(np.abs(z).sum(axis=1) <= R)
        se = math.sqrt(p * (1 - p) / z.shape[0])
        assert abs(rfd.l1_ball_mass(R) - p) < 5 * se


def test_c_r_direct_triple_integral():
    # Independent route: the full-space triple integral over the octahedron.
    R = 1.5
    phi = lambda t: math.exp(-0.5 * t * t) / math.sqrt(2 * math.pi)
    val, _ = scipy.integrate.tplquad(
        lambda c, b, a: phi(a) * phi(b) * phi(c),
        -R, R,
        lambda a: -(R - abs(a)), lambda a: R - abs(a),
        lambda a, b: -(R - abs(a) - abs(b)), lambda a, b: R - abs(a) - abs(b),
        epsabs=1e-12, epsrel=1e-10)
    assert rfd.l1_ball_mass(R) == pytest.approx(val, rel=1e-8)


def test_c_r_default_radius_tail():
    # 1 - C_10 ~ 3.1e-8 (SURVEY [S7], nested quadrature; chi-square bound 2.7e-7).
    pin = PINS["c_r_tail_R10"]
    assert 1.0 - C_R == pytest.approx(pin["value"], rel=pin["rel_tol"])
    assert 0 < 1.0 - C_R < 2.7e-7


# ---------------------------------------------------------------- a1: omega
def test_frequency_anchor_seed0():
    # SURVEY.md Sec. 8(c) pins: seed 0 -> omega_0 after fp32 rounding.
    om, att = rfd.frequencies(0, 4)
    pin = PINS["omega0_seed0"]
    np.testing.assert_allclose(om[0], pin["value"], rtol=0, atol=pin["abs_tol"])
    assert att[0] == 1


def test_frequencies_every_config_seed():
    # SURVEY.md [S12] (tests/golden/pins.json "config_seed_frequencies"): for
    # each config seed, the nu range and max|omega_c| over all m frequencies
    # and no rejections.  Covers every frequency of every seed (a swapped
    # (k, attempt) counter word or key word would change them).
    pin = PINS["config_seed_frequencies"]
    for row in pin["rows"]:
        om, att = rfd.frequencies(row["seed"], row["m"])
        nu = rfd.importance_weights(om, row["eps"], C_R)
        assert att.max() == 1, row
        assert nu.min() == pytest.approx(row["nu_min"], rel=pin["rel_tol"]), row
        assert nu.max() == pytest.approx(row["nu_max"], rel=pin["rel_tol"]), row
        assert float(np.abs(om).max()) == pytest.approx(row["max_abs_omega"], abs=pin["abs_tol_omega"])


def test_estimator_unbiased_at_coincident_and_far_points():
    # SPEC.md:390-398 (build_decomposition examples, DERIVED by Monte Carlo):
    # over 50 seeds the RF estimate W~(v, w) = (1/m) sum cos(2 pi omega.z)
    # tau/p has mean within 3 standard errors of f(z):
    # 1 for coincident points, 0 at distance 2 eps.  At z = (eps, eps, 0) --
    # L1 distance 2 eps, but a corner of the L-infinity cube -- the Fourier
    # inversion of the product-sinc converges to the corner value 1/2 * 1/2 =
    # 1/4, not 0: the estimator targets the cube graph (A2).
    eps, m = 0.15, 256
    for z, want in (([0.0, 0.0, 0.0], 1.0), ([2 * eps, 0.0, 0.0], 0.0),
                    ([eps, eps, 0.0], 0.25)):
        vals = np.array([rfd.estimator(np.array([z]), rfd.frequencies(5000 + s, m)[0], eps, C_R)[0]
                         for s in range(50)])
        se = vals.std(ddof=1) / math.sqrt(vals.size)
        assert abs(vals.mean() - want) < 3 * se, (z, vals.mean(), se)


def test_frequencies_truncated_and_gaussian():
    om, att = rfd.frequencies(99, 4096)
    assert np.all(np.abs(om.astype(np.float64)).sum(axis=1) <= rfd.DEFAULT_R + 1e-5)
    m = om.shape[0]
    assert np.all(np.abs(om.mean(axis=0)) <= 4 / math.sqrt(m))
    assert np.all(np.abs(om.var(axis=0) - 1.0) < 0.08)
    for c in range(3):
        assert scipy.stats.kstest(om[:, c], "norm").pvalue > 1e-3


def test_frequencies_small_radius_rejects():
    om, att = rfd.frequencies(5, 256, R=1.5)
    assert np.all(np.abs(om.astype(np.float64)).sum(axis=1) <= 1.5 + 1e-6)
    assert att.max() > 1


def test_frequencies_deterministic_and_prefix_stable():
    a, _ = rfd.frequencies(3, 64)
    b, _ = rfd.frequencies(3, 128)
    np.testing.assert_array_equal(a, b[:64])


# ---------------------------------------------------------------- a3: features
def test_features_unit_modulus_and_estimator_form():
    rng = np.random.default_rng(0)
    X = rng.random((40, 3)).astype(np.float32)
    om, _ = rfd.frequencies(11, 24)
    eps = 0.2
    nu = rfd.importance_weights(om, eps, C_R)
    P = rfd.features(X, om)
    m = om.shape[0]
    np.testing.assert_allclose(P[:, :m] ** 2 + P[:, m:] ** 2, 1.0, atol=1e-15)
    W = P @ (np.concatenate([nu, nu])[:, None] * P.T)
    # The paper's estimator on z = x_v - x_w.
    for v, w in ((0, 1), (3, 3), (7, 30)):
        z = X[v].astype(np.float64) - X[w].astype(np.float64)
        assert W[v, w] == pytest.approx(rfd.estimator(z[None, :], om, eps, C_R)[0], rel=1e-12, abs=1e-14)
    # W~_ii = sum nu (a per-plan constant).
    np.testing.assert_allclose(np.diag(W), nu.sum(), rtol=1e-13)


# ---------------------------------------------------------------- a4, a6
def _brute_features(x, om):
    row = [math.cos(2 * math.pi * sum(float(o[c]) * float(x[c]) for c in range(3))) for o in om]
    row += [math.sin(2 * math.pi * sum(float(o[c]) * float(x[c]) for c in range(3))) for o in om]
    return row


def test_gram_brute_force_and_trace():
    rng = np.random.default_rng(1)
    X = rng.random((37, 3)).astype(np.float32)
    om, _ = rfd.frequencies(2, 6)
    r = 12
    G = rfd.gram(X, om, chunk=10)
    Gb = [[0.0] * r for _ in range(r)]
    for x in X:
        f = _brute_features(x, om)
        for a in range(r):
            for b in range(r):
                Gb[a][b] += f[a] * f[b]
    np.testing.assert_allclose(G, np.array(Gb), rtol=1e-12, atol=1e-12)
    # Trace identity: sum_k G_cc,kk + G_ss,kk = N m.
    assert np.trace(G) == pytest.approx(37 * 6, rel=1e-14)
    assert np.allclose(G, G.T)
    assert np.linalg.eigvalsh(G).min() > -1e-10


def test_project_brute_force_unit_and_linearity():
    rng = np.random.default_rng(2)
    X = rng.random((29, 3)).astype(np.float32)
    om, _ = rfd.frequencies(4, 5)
    F = rng.standard_normal((29, 3))
    S = rfd.project(X, om, F, chunk=7)
    Sb = np.zeros((10, 3))
    for i, x in enumerate(X):
        Sb += np.outer(_brute_features(x, om), F[i])
    np.testing.assert_allclose(S, Sb, rtol=1e-12, atol=1e-12)
    e = np.zeros((29, 1))
    e[13] = 1.0
    np.testing.assert_allclose(rfd.project(X, om, e)[:, 0], _brute_features(X[13], om), atol=1e-15)
    F2 = rng.standard_normal((29, 3))
    np.testing.assert_allclose(rfd.project(X, om, 2 * F - 3 * F2),
                               2 * S - 3 * rfd.project(X, om, F2), atol=1e-12)


# ---------------------------------------------------------------- a5: core
def test_phi1_spec_examples():
    # SPEC.md:414-416.
    r = 5
    np.testing.assert_allclose(rfd.phi1_lam(np.zeros((r, r)), 0.7), 0.7 * np.eye(r), atol=1e-15)
    np.testing.assert_allclose(rfd.phi1_lam(np.eye(r), 1.0), (math.e - 1) * np.eye(r), rtol=1e-13)
    rng = np.random.default_rng(3)
    M = rng.standard_normal((8, 8))
    lam = -0.6
    ref = scipy.linalg.solve(M.T, (scipy.linalg.expm(lam * M) - np.eye(8)).T).T
    np.testing.assert_allclose(rfd.phi1_lam(M, lam), ref, rtol=1e-10, atol=1e-12)


def test_phi1_rank1_spec_example():
    # A = B = e1 (N = 2, one column), Lambda = 1, X = [1, 1] -> [e, 1].
    A = np.array([[1.0], [0.0]])
    X = np.array([1.0, 1.0])
    out = X + A @ (rfd.phi1_lam(A.T @ A, 1.0) @ (A.T @ X))
    np.testing.assert_allclose(out, [math.e, 1.0], rtol=1e-14)


def test_core_zero_lambda_and_diagonal_closed_form():
    rng = np.random.default_rng(4)
    m = 4
    g = rng.uniform(0.5, 3.0, 2 * m)
    nu = rng.uniform(0.01, 0.2, m)
    np.testing.assert_array_equal(rfd.core(np.diag(g), nu, 0.0), np.zeros((2 * m, 2 * m)))
    lam = -1.3
    d = np.concatenate([nu, nu])
    C = rfd.core(np.diag(g), nu, lam)
    np.testing.assert_allclose(np.diag(C), np.expm1(lam * g * d) / g, rtol=1e-13)
    assert np.abs(C - np.diag(np.diag(C))).max() < 1e-15


def test_core_symmetric():
    rng = np.random.default_rng(5)
    X = rng.random((200, 3)).astype(np.float32)
    om, _ = rfd.frequencies(6, 16)
    nu = rfd.importance_weights(om, 0.1, C_R)
    C = rfd.core(rfd.gram(X, om), nu, -0.9)
    assert np.abs(C - C.T).max() <= 1e-12 * np.abs(C).max()


def test_proposal_pdf_normalised_on_ball():
    # int_{B(R)} p = 1 by direct triple quadrature (pins (2 pi)^{-3/2} / C_R of
    # PAPER.md:936), at a radius where the integrand is well resolved.
    R = 2.5
    c = rfd.l1_ball_mass(R)
    p = lambda a, b, cc: float(rfd.proposal_pdf(np.array([a, b, cc]), c))
    val, _ = scipy.integrate.tplquad(
        lambda cc, b, a: p(a, b, cc), -R, R,
        lambda a: -(R - abs(a)), lambda a: R - abs(a),
        lambda a, b: -(R - abs(a) - abs(b)), lambda a, b: R - abs(a) - abs(b),
        epsabs=1e-11, epsrel=1e-9)
    assert val == pytest.approx(1.0, rel=1e-7)


def test_importance_weights_definition_pieces():
    om, _ = rfd.frequencies(8, 32)
    eps = 0.12
    nu = rfd.importance_weights(om, eps, C_R)
    k = 5
    w = om[k].astype(np.float64)
    tau_k = np.prod([math.sin(2 * math.pi * eps * c) / (math.pi * c) for c in w])
    p_k = math.exp(-0.5 * float(w @ w)) / ((2 * math.pi) ** 1.5 * C_R)
    assert nu[k] == pytest.approx(tau_k / (32 * p_k), rel=1e-13)
