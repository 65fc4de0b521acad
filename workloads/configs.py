"""Input generators for BASELINE.json ``configs`` (recipes: SURVEY.md Sec. 8(d)).

The paper measures on Thingi10K meshes, barycenter meshes, ModelNet10 clouds
and random 3-D sets; none are in the
container.  These seeded synthetic inputs stand in for them at matching
scales.  Each generator uses ``numpy.random.default_rng``
(PCG64) with the config seed; outputs are fp32, row-major.  The plan seed of
each config equals its input seed.

No RFD arithmetic lives here.
"""

import math

import numpy as np


def _sphere(rng, n):
    g = rng.standard_normal((n, 3))
    return g / np.linalg.norm(g, axis=1, keepdims=True)


def cfg1(n=1024):
    """N=1024 uniform on the unit sphere, F N x 3 iid N(0,1)."""
    rng = np.random.default_rng(0)
    x = _sphere(rng, n)
    F = rng.standard_normal((n, 3))
    return x.astype(np.float32), F.astype(np.float32)


def cfg2(n=8192):
    """Torus R=1, r=0.3 uniform by area, jitter N(0, 0.005^2); smooth field."""
    rng = np.random.default_rng(1)
    us, vs = [], []
    while sum(len(v) for v in vs) < n:
        u = rng.uniform(0.0, 2.0 * math.pi, n)
        v = rng.uniform(0.0, 2.0 * math.pi, n)
        keep = rng.uniform(0.0, 1.0, n) < (1.0 + 0.3 * np.cos(v)) / 1.3
        us.append(u[keep])
        vs.append(v[keep])
    u = np.concatenate(us)[:n]
    v = np.concatenate(vs)[:n]
    x = np.stack([(1.0 + 0.3 * np.cos(v)) * np.cos(u),
                  (1.0 + 0.3 * np.cos(v)) * np.sin(u),
                  0.3 * np.sin(v)], axis=1)
    x = x + rng.normal(0.0, 0.005, x.shape)
    base = np.sin(3.0 * x[:, 0]) + np.cos(2.0 * x[:, 1]) + x[:, 2]
    F = base[:, None] + rng.normal(0.0, 0.1, (n, 3))
    return x.astype(np.float32), F.astype(np.float32)


def _rotation(rng):
    q, r = np.linalg.qr(rng.standard_normal((3, 3)))
    return q * np.sign(np.diag(r))[None, :]


def cfg3(clouds=256, n=2048, applications=50):
    """256 ellipsoid clouds x 2048 points, unit-cube normalised; 50 Dirichlet(1)
    vectors per cloud (v_0 = the cloud's weights, v_t from rng (2, cloud, t)).

    Returns x (clouds, n, 3) and V (applications, clouds, n, 1).
    """
    rng = np.random.default_rng(2)
    xs = np.empty((clouds, n, 3))
    V = np.empty((applications, clouds, n, 1))
    for c in range(clouds):
        axes = rng.uniform(0.3, 1.0, 3)
        p = _sphere(rng, n) * axes[None, :]
        p = p @ _rotation(rng).T
        lo = p.min(axis=0)
        p = (p - lo) / np.max(p.max(axis=0) - lo)
        xs[c] = p
        V[0, c, :, 0] = rng.dirichlet(np.ones(n))
    for c in range(clouds):
        for t in range(1, applications):
            V[t, c, :, 0] = np.random.default_rng((2, c, t)).dirichlet(np.ones(n))
    return xs.astype(np.float32), V.astype(np.float32)


def cfg4(n=200_000):
    """Deformed sheet z = 0.1 sin(4x) cos(4y) on [0,1)^2, jitter N(0, 0.002^2)."""
    rng = np.random.default_rng(3)
    xy = rng.uniform(0.0, 1.0, (n, 2))
    z = 0.1 * np.sin(4.0 * xy[:, 0]) * np.cos(4.0 * xy[:, 1])
    x = np.concatenate([xy, z[:, None]], axis=1)
    x = x + rng.normal(0.0, 0.002, x.shape)
    F = rng.standard_normal((n, 3))
    return x.astype(np.float32), F.astype(np.float32)


def cfg5(n=4_194_304, d=16):
    """N = 2^22 iid uniform in the unit cube, F N x 16 iid N(0,1)."""
    rng = np.random.default_rng(4)
    x = rng.random((n, 3), dtype=np.float32)
    F = rng.standard_normal((n, d), dtype=np.float32)
    return x, F


# Parameters per config (BASELINE.json ``configs``).
CONFIGS = {
    1: dict(name="cfg1_sphere", eps=0.15, lam=-0.5, m=16, seed=0, d=3, n=1024),
    2: dict(name="cfg2_torus", eps=0.08, lam=-1.0, m=64, seed=1, d=3, n=8192),
    3: dict(name="cfg3_ellipsoids", eps=0.1, lam=-2.0, m=32, seed=2, d=1,
            n=2048, clouds=256, applications=50),
    4: dict(name="cfg4_sheet", eps=0.02, lam=-0.8, m=128, seed=3, d=3, n=200_000),
    5: dict(name="cfg5_cube", eps=0.01, lam=-0.3, m=256, seed=4, d=16,
            n=4_194_304),
}

_GEN = {1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4, 5: cfg5}


def make_config(cfg, **overrides):
    """(params dict, x, F) for a config; ``overrides`` are passed to the generator
    (e.g. n=65536 for a bounded sample of cfg 5)."""
    params = dict(CONFIGS[cfg])
    x, F = _GEN[cfg](**overrides)
    if cfg == 3:
        params["clouds"], params["n"] = x.shape[0], x.shape[1]
        params["applications"] = F.shape[0]
    else:
        params["n"] = x.shape[0]
    return params, x, F


def barycenter_inputs(n=2000, floor=0.0, width=0.5, k=3, seed=7):
    """Alg. 1 inputs (k = 3 distributions "with mass
    concentrated in vertices surrounding a distinct center vertex", area
    weights): n uniform sphere points, uniform area weights a = 1/n, and k
    Gaussian bumps of width `width` around points 0..k-1 plus a constant
    `floor`, each normalised to <a, mu^i> = 1.  Returns (x fp32 n x 3, a fp64
    n, mus fp64 k x n)."""
    rng = np.random.default_rng(seed)
    x = _sphere(rng, n).astype(np.float32)
    a = np.full(n, 1.0 / n)
    xd = x.astype(np.float64)
    mus = np.stack([np.exp(-((xd - xd[i]) ** 2).sum(1) / (2 * width ** 2)) + floor
                    for i in range(k)])
    mus /= (mus @ a)[:, None]
    return x, a, mus
