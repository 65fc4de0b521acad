"""Pins for oracle/dense.py: the exact epsilon-NN graph diffusion on tiny N
(Eq. 4 at PAPER.md:128-133; Eq. 9 at PAPER.md:286-295),
a diagnostic (never a parity gate) -- no GPU."""

import math

import numpy as np
import scipy.linalg

from oracle import dense


def test_dense_spec_examples():
    # SPEC.md:199-201.
    X = np.eye(3)
    np.testing.assert_allclose(dense.symmetric_expm_apply(np.eye(3), 1.0, X), math.e * X, rtol=1e-14)
    np.testing.assert_allclose(
        dense.symmetric_expm_apply(np.diag([0.0, math.log(2.0)]), 1.0, np.ones(2))[:, 0],
        [1.0, 2.0], rtol=1e-14)
    rng = np.random.default_rng(0)
    A = rng.standard_normal((30, 30))
    W = A + A.T
    np.testing.assert_allclose(dense.symmetric_expm_apply(W, 0.1, np.eye(30)),
                               scipy.linalg.expm(0.1 * W), rtol=1e-10, atol=1e-12)


def test_dense_graph_two_points():
    X = np.array([[0.0, 0.0, 0.0], [0.1, 0.1, 0.0]])
    # L-inf distance 0.1 <= 0.15 but L1 distance 0.2 > 0.15.
    assert dense.epsilon_graph(X, 0.15, "inf")[0, 1] == 1.0
    assert dense.epsilon_graph(X, 0.15, 1)[0, 1] == 0.0
    np.testing.assert_allclose(dense.exact_diffusion(X, np.eye(2), 0.15, 1.0, 1), np.eye(2) * math.e,
                               rtol=1e-14)


def test_two_points_within_eps_closed_form():
    # A = [[1, 1], [1, 1]] (unit diagonal, A4): eigenvalues 0 and 2,
    # so exp(lam A) = I + (e^{2 lam} - 1)/2 J.
    X = np.array([[0.0, 0.0, 0.0], [0.05, -0.1, 0.02]])
    F = np.array([[1.0, -2.0], [3.0, 0.5]])
    lam = -0.7
    want = F + 0.5 * math.expm1(2 * lam) * np.ones((2, 2)) @ F
    for norm in ("inf", 1):
        np.testing.assert_allclose(dense.exact_diffusion(X, F, 0.2, lam, norm), want, rtol=1e-13)


def test_path_graph_and_inclusive_boundary():
    # Three points on a line at spacing eps: edges 0-1 and 1-2 only (the
    # boundary is inclusive, A11; 0-2 is at 2 eps), i.e. A = I + path(3),
    # whose exp is known in closed form from the path's eigenvalues 0, +-sqrt 2.
    eps = 0.25
    X = np.array([[0.0, 0.0, 0.0], [eps, 0.0, 0.0], [2 * eps, 0.0, 0.0]])
    A = dense.epsilon_graph(X, eps, "inf")
    np.testing.assert_array_equal(A, [[1, 1, 0], [1, 1, 1], [0, 1, 1]])
    lam = 0.3
    r2 = math.sqrt(2.0)
    v = [np.array([1, r2, 1]) / 2, np.array([1, 0, -1]) / r2, np.array([1, -r2, 1]) / 2]
    ev = [1 + r2, 1.0, 1 - r2]
    K = sum(math.exp(lam * e) * np.outer(u, u) for e, u in zip(ev, v))
    np.testing.assert_allclose(dense.exact_diffusion(X, np.eye(3), eps, lam), K, rtol=1e-13)
    np.testing.assert_allclose(K, scipy.linalg.expm(lam * A), rtol=1e-13)


def test_sparse_route_matches_dense():
    # the sparse graph (cKDTree pairs) and expm_multiply against the dense
    # brute-force graph and eigh route, both norms, including boundary pairs
    rng = np.random.default_rng(4)
    X = rng.random((300, 3))
    X[1] = X[0] + np.array([0.1, 0.0, 0.0])  # exactly at eps in both norms (A11: inclusive)
    F = rng.standard_normal((300, 2))
    for norm in ("inf", 1):
        A = dense.epsilon_graph(X, 0.1, norm)
        As = dense.epsilon_graph_sparse(X, 0.1, norm).toarray()
        np.testing.assert_array_equal(As, A)
        np.testing.assert_allclose(dense.exact_diffusion_sparse(X, F, 0.1, -0.7, norm),
                                   dense.exact_diffusion(X, F, 0.1, -0.7, norm), rtol=1e-10, atol=1e-12)
