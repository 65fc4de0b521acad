"""The spread-grid identity behind a4's large-cloud path (k_nufft.cu,
DESIGN.md Sec. 6 "a4 spread grid"), checked in fp64 numpy on the CPU against
the oracle's direct sum G = Phi^T Phi.

This pins the *method* the GPU kernels implement -- kernel width, beta,
grid spacing rule, deconvolution and the G assembly from the grid Gram --
independently of the CUDA code (restated here, not imported); the GPU result
itself is gated against the oracle in tests/test_gpu_parity.py
(test_gram_spread_grid_parity).
"""
import math

import numpy as np
import pytest

from oracle import rfd as orf
from workloads import make_config


def _es(z, beta):
    out = np.zeros_like(z)
    msk = np.abs(z) < 1.0
    out[msk] = np.exp(beta * (np.sqrt(1.0 - z[msk] ** 2) - 1.0))
    return out


def _phihat(s, alpha, beta, nq=200):
    # phi^(s) = int psi(x / alpha) e^{i s x} dx = alpha int_{-1}^{1} psi(z) cos(s alpha z) dz
    z, wq = np.polynomial.legendre.leggauss(nq)
    return alpha * (np.cos(np.outer(s, alpha * z)) @ (wq * _es(z, beta)))


def spread_grid_gram(X, omega, w=8, hfac=1.5):
    """G through the spread grid, following the kernels' parameter rules."""
    beta = 2.30 * w
    lo, hi = X.min(0), X.max(0)
    c = lo + 0.5 * (hi - lo)
    Y = X - c
    Xh = np.abs(Y).max(0) * (1 + 1e-6) + 1e-30
    S = np.maximum(4.0 * math.pi * np.abs(omega).max(0), 1e-3)
    ht = hfac / S
    e = np.floor(np.log2(ht)) - 3
    h = np.floor(ht / 2.0 ** e) * 2.0 ** e          # q 2^e, 8 <= q < 16
    alpha = 0.5 * w * h
    L = (np.ceil((Xh + alpha) / h) + 1).astype(int)
    n = 2 * L + 1
    b = np.zeros(tuple(n))
    idx, vals = [], []
    for a in range(3):
        cell = np.floor(Y[:, a] / h[a]).astype(int)      # [l h, (l + 1) h)
        ls = cell[:, None] + np.arange(-w // 2 + 1, w // 2 + 1)[None, :]
        vals.append(_es((ls * h[a] - Y[:, a:a + 1]) / alpha[a], beta))
        idx.append(ls + L[a])
    for i in range(w):
        for j in range(w):
            vxy = vals[0][:, i] * vals[1][:, j]
            for k in range(w):
                np.add.at(b, (idx[0][:, i], idx[1][:, j], idx[2][:, k]), vxy * vals[2][:, k])
    nodes = np.stack(np.meshgrid(*[(np.arange(n[a]) - L[a]) * h[a] for a in range(3)],
                                 indexing="ij"), -1).reshape(-1, 3)
    bw = b.reshape(-1)
    th = 2.0 * math.pi * nodes @ omega.T
    C, Sn = np.cos(th), np.sin(th)
    Tcc, Tss = (C * bw[:, None]).T @ C, (Sn * bw[:, None]).T @ Sn
    Tsc, Tcs = (Sn * bw[:, None]).T @ C, (C * bw[:, None]).T @ Sn
    m = omega.shape[0]
    sp = 2.0 * math.pi * (omega[:, None, :] + omega[None, :, :])
    sm = 2.0 * math.pi * (omega[:, None, :] - omega[None, :, :])
    dp, dm = np.ones((m, m)), np.ones((m, m))
    for a in range(3):
        dp *= _phihat(sp[..., a].ravel(), alpha[a], beta).reshape(m, m) / h[a]
        dm *= _phihat(sm[..., a].ravel(), alpha[a], beta).reshape(m, m) / h[a]
    Pp = ((Tcc - Tss) + 1j * (Tsc + Tcs)) / dp     # Psi(omega_j + omega_k)
    Pm = ((Tcc + Tss) + 1j * (Tsc - Tcs)) / dm     # Psi(omega_j - omega_k)
    G = np.empty((2 * m, 2 * m))
    G[:m, :m] = 0.5 * (Pm.real + Pp.real)
    G[m:, m:] = 0.5 * (Pm.real - Pp.real)
    G[:m, m:] = 0.5 * (Pp.imag - Pm.imag)
    G[m:, :m] = 0.5 * (Pp.imag + Pm.imag)
    return G, c, int(np.prod(n))


@pytest.mark.parametrize("cfg,n,m", [(5, 16384, 64), (4, 20000, 32), (2, None, 32)])
def test_spread_grid_identity_reproduces_direct_gram(cfg, n, m):
    p, x, _ = make_config(cfg, **({"n": n} if n else {}))
    X = np.asarray(x, np.float64)
    omega = np.asarray(orf.frequencies(p["seed"], m)[0])
    G, c, nodes = spread_grid_gram(X, omega)
    Gd = orf.gram(X - c, omega)              # the centred basis the library works in
    err = np.abs(G - Gd).max() / np.abs(Gd).max()
    assert err <= 3e-6, (err, nodes)  # (the GPU's direct fp16 hi/lo Gram: ~5e-6)
    np.testing.assert_allclose(G, G.T, rtol=0, atol=1e-9 * np.abs(Gd).max())


def test_spread_grid_width_matters():
    # the error falls with the kernel width (a dropped deconvolution factor or
    # a wrong grid spacing would not behave like this)
    p, x, _ = make_config(5, n=4096)
    X = np.asarray(x, np.float64)
    omega = np.asarray(orf.frequencies(p["seed"], 32)[0])
    errs = []
    for w in (4, 8):
        G, c, _ = spread_grid_gram(X, omega, w=w)
        Gd = orf.gram(X - c, omega)
        errs.append(np.abs(G - Gd).max() / np.abs(Gd).max())
    assert errs[1] < errs[0] / 10, errs
