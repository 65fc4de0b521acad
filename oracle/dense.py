"""Exact epsilon-NN graph diffusion on tiny N (diagnostic, not a parity gate).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Brute force of PAPER.md:80 ("calculate a kernel matrix K ... then matrix
vector multiplications") for the graph diffusion kernel K = exp(lambda W_G)
(Eq. 4) of the epsilon-NN graph (Eq. 9,
f(z) = 1[||z|| <= eps]) with binary weights and a unit diagonal, f(0) = 1
(A4, A11).  The method's tau is the transform of the L-infinity
ball (A2), so ``norm="inf"`` is the primary ground truth and
``norm=1`` (the norm the paper names) a labelled secondary.

Pins: eigh-based exp against scipy.linalg.expm on random symmetric input and
the closed forms of SPEC.md:199-203, two-point and path-graph closed forms
(tests/test_oracle_dense.py).  The RFD
approximation error against this graph is parity unpinned (no paper value
for synthetic inputs); it is reported, never gated.
"""

import numpy as np


def epsilon_graph(X, eps, norm="inf"):
    """A_ij = 1[||x_i - x_j|| <= eps] (inclusive; unit diagonal), fp64 distances."""
    X = np.asarray(X, np.float64)
    diff = X[:, None, :] - X[None, :, :]
    if norm == "inf":
        dist = np.max(np.abs(diff), axis=-1)
    elif norm == 1:
        dist = np.sum(np.abs(diff), axis=-1)
    else:
        raise ValueError("norm must be 'inf' or 1")
    return (dist <= eps).astype(np.float64)


def symmetric_expm_apply(W, lam, F):
    """exp(lam W) F for symmetric W via W = Q diag(w) Q^T."""
    W = np.asarray(W, np.float64)
    w, Q = np.linalg.eigh(W)
    F = np.asarray(F, np.float64)
    return Q @ (np.exp(lam * w)[:, None] * (Q.T @ F.reshape(W.shape[0], -1)))


def exact_diffusion(X, F, eps, lam, norm="inf"):
    """Brute-force GFI i = exp(lam A) F on the exact epsilon-graph."""
    return symmetric_expm_apply(epsilon_graph(X, eps, norm), lam, F)


def epsilon_graph_sparse(X, eps, norm="inf"):
    """The same graph as ``epsilon_graph`` as a scipy.sparse CSR matrix (unit
    diagonal, inclusive boundary: cKDTree.query_pairs returns pairs at
    distance <= eps in the Minkowski p-norm, p = inf or 1), for N beyond the
    dense route (cfg 2: 8192 points)."""
    import scipy.sparse
    import scipy.spatial
    X = np.asarray(X, np.float64)
    n = X.shape[0]
    p = np.inf if norm == "inf" else 1
    if norm not in ("inf", 1):
        raise ValueError("norm must be 'inf' or 1")
    pairs = scipy.spatial.cKDTree(X).query_pairs(eps, p=p, output_type="ndarray")
    i = np.concatenate([pairs[:, 0], pairs[:, 1], np.arange(n)])
    j = np.concatenate([pairs[:, 1], pairs[:, 0], np.arange(n)])
    return scipy.sparse.csr_matrix((np.ones(i.size), (i, j)), shape=(n, n))


def exact_diffusion_sparse(X, F, eps, lam, norm="inf"):
    """exp(lam A) F on the sparse exact epsilon-graph (scipy's expm_multiply,
    a library primitive: the action of the matrix exponential)."""
    import scipy.sparse.linalg
    A = epsilon_graph_sparse(X, eps, norm)
    F = np.asarray(F, np.float64).reshape(A.shape[0], -1)
    return scipy.sparse.linalg.expm_multiply(lam * A, F)
