"""RFDiffusion (RFD) integrator, step by step, in fp64 on the CPU.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  The product path must
never import this module.

What it computes (Sec. 2.4 "RFDiffusion", lines 283-366, and
Appendix A.4):

    out = exp(lambda * W~) F,   W~ = Phi D Phi^T  (N x N, never formed)

with the closed form of PAPER.md:327-339 / Eq. 13 written
inverse-free (reading A5):

    out = F + Phi . C^ . (Phi^T F),   C^ = lambda * D * phi1(lambda * G * D),
    G = Phi^T Phi,  phi1(Z) = sum_k Z^k / (k+1)!.

Step order:
  a1 ``frequencies``      omega_k ~ N(0, I_3) truncated to ||omega||_1 <= R
  a2 ``importance_weights`` nu_k = tau(omega_k) / (m p(omega_k))
  a3 ``features``         phi(x) = [cos 2 pi omega_k.x ; sin 2 pi omega_k.x]
  a4 ``gram``             G = Phi^T Phi
  a5 ``core``             C^ = D * (top-right block of expm([[lam G D, lam I],[0,0]]))
  a6 ``project``          S = Phi^T F
  a7                      Y = C^ S
  a8                      out = F + Phi Y

The only grouping not written in the paper: sums over points (G, S) and the
row-wise pass a8 are evaluated over consecutive chunks of ``CHUNK`` points so
that Phi (17 GB at N = 4M, m = 256) is never held whole.  Each chunk's
contribution is a library matmul; chunk sums are added in point order.

Pins (tests/test_oracle_rfd.py, tests/test_oracle_integrator.py):
  * a1: stream words pinned via oracle.philox (curand KAT); truncation
    invariant; Gaussian moments; SURVEY anchor omega_0 for seed 0.
  * a2: tau(0) = (2 eps)^3; SPEC value -1.24732 at eps = 1, omega = (.6,0,0)
    (SPEC.md:380); 1-D quadrature of the indicator's Fourier integral;
    C_R against an independent Monte-Carlo / nquad estimate.
  * a3: Phi D Phi^T equals the paper's own estimator form
    (1/m) sum_k cos(2 pi omega_k^T z) tau/p.
  * a4: trace identity sum_k G_cc,kk + G_ss,kk = N m; brute-force loop.
  * a5: phi1 special cases; diagonal closed form.
  * whole: identity against dense expm of the same low-rank matrix; N = 1
    and N = 2 closed forms; lambda -> 0; semigroup; symmetry; linearity;
    permutation equivariance.
  * approximation quality against the exact epsilon-graph: parity unpinned
    (the paper prints no values for synthetic inputs); trend test only.
"""

import concurrent.futures
import math
import os

import numpy as np
import scipy.integrate
import scipy.linalg
import scipy.special
import threadpoolctl

from . import philox

# Counter word 2 of every Philox call that draws a frequency (A14).
FREQ_TAG = 0x52464421
# L1 truncation radius of the Gaussian proposal (A6).
DEFAULT_R = 10.0
# Rejection attempts per frequency before giving up (P(reject) = 3.1e-8).
MAX_ATTEMPTS = 64
# Points per chunk for sums over points (memory only; see module docstring).
CHUNK = 65536


# --------------------------------------------------------------------------
# a1  frequencies
# --------------------------------------------------------------------------
def frequencies(seed, m, R=DEFAULT_R):
    """Draw omega_1..omega_m iid from N(0, I_3) truncated to the L1 ball B(R).

    PAPER.md:316 ("Take omega_1, ..., omega_m iid ~ P"), PAPER.md:323 ("Here
    we use (truncated) Gaussian"), PAPER.md:374 and 936 (Gaussian truncated to
    the L1-ball B(R), sigma = 1).  Stream layout (A14): for
    frequency k and attempt a, Philox4x32-10 with counter (k, a, TAG, 0) and
    key (seed lo, seed hi) gives words w0..w3; u_j = (w_j + 0.5) 2^-32;
    Box-Muller z0 = sqrt(-2 ln u0) cos 2 pi u1, z1 = sqrt(-2 ln u0) sin 2 pi u1,
    z2 = sqrt(-2 ln u2) cos 2 pi u3; accept iff |z0|+|z1|+|z2| <= R; the
    accepted z is rounded once to fp32.

    Returns (omega float32 (m, 3), attempts int (m,)).
    """
    seed = int(seed)
    key = (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    omega = np.zeros((m, 3), dtype=np.float32)
    attempts = np.zeros(m, dtype=np.int64)
    for k in range(m):
        for a in range(MAX_ATTEMPTS):
            w = philox.philox4x32_10((k, a, FREQ_TAG, 0), key)
            u = [(wj + 0.5) * 2.0 ** -32 for wj in w]
            r01 = math.sqrt(-2.0 * math.log(u[0]))
            r23 = math.sqrt(-2.0 * math.log(u[2]))
            z = (r01 * math.cos(2.0 * math.pi * u[1]),
                 r01 * math.sin(2.0 * math.pi * u[1]),
                 r23 * math.cos(2.0 * math.pi * u[3]))
            if abs(z[0]) + abs(z[1]) + abs(z[2]) <= R:
                omega[k] = np.array(z, dtype=np.float64).astype(np.float32)
                attempts[k] = a + 1
                break
        else:
            raise RuntimeError("frequency %d: no accepted draw in %d attempts"
                               % (k, MAX_ATTEMPTS))
    return omega, attempts


# --------------------------------------------------------------------------
# a2  importance weights
# --------------------------------------------------------------------------
def l1_ball_mass(R=DEFAULT_R):
    """C_R = P(||Z||_1 <= R) for Z ~ N(0, I_3): the normaliser of the truncated pdf.

    PAPER.md:385 (C = int_{B(R)} (2 pi)^{-3/2} exp(-||r||^2 / 2) dr) and 936.
    Written out: by symmetry over the 8 octants,
        C_R = int_0^R int_0^{R-a} h(a) h(b) erf((R-a-b)/sqrt 2) db da,
    h(t) = 2 exp(-t^2/2)/sqrt(2 pi) (the half-normal density) and
    P(|Z_3| <= s) = erf(s / sqrt 2).  DESIGN.md A7.
    """
    def h(t):
        return 2.0 * math.exp(-0.5 * t * t) / math.sqrt(2.0 * math.pi)

    def inner(b, a):
        return h(a) * h(b) * math.erf((R - a - b) / math.sqrt(2.0))

    val, _ = scipy.integrate.dblquad(inner, 0.0, R, lambda a: 0.0,
                                     lambda a: R - a, epsabs=1e-15,
                                     epsrel=1e-13)
    return val


def tau(omega, eps):
    """Fourier transform of the epsilon-box indicator, product of 1-D sincs.

    PAPER.md:361-366 prints tau(xi) = prod_i sin(2 eps xi_i) / xi_i.  Under
    the paper's own convention f(z) = int exp(2 pi i omega^T z) tau(omega)
    d omega the 1-D factor is sin(2 pi eps w) / (pi w), with
    limit 2 eps at w = 0 (A1).  The product of 1-D factors is the
    transform of the L-infinity (cube) indicator (A2).
    """
    w = np.asarray(omega, dtype=np.float64)
    fac = np.empty_like(w)
    nz = w != 0.0
    fac[nz] = np.sin(2.0 * math.pi * eps * w[nz]) / (math.pi * w[nz])
    fac[~nz] = 2.0 * eps
    return np.prod(fac, axis=-1)


def proposal_pdf(omega, c_r):
    """pdf of the R-truncated standard Gaussian on R^3.

    p(omega) = (2 pi)^{-3/2} exp(-||omega||^2 / 2) / C_R.
    """
    w = np.asarray(omega, dtype=np.float64)
    return (2.0 * math.pi) ** -1.5 * np.exp(-0.5 * np.sum(w * w, axis=-1)) / c_r


def importance_weights(omega, eps, c_r):
    """nu_k = tau(omega_k) / (m p(omega_k)).

    PAPER.md:316-319: nu_i = sqrt(tau / p) on each side with a 1/sqrt(m)
    prefactor on each side; in the real two-column form the product of both
    sides, tau / (m p), sits in D = diag(nu, nu) (A3;
    SPEC.md:363).
    """
    m = np.asarray(omega).shape[0]
    return tau(omega, eps) / (m * proposal_pdf(omega, c_r))


# --------------------------------------------------------------------------
# a3  features
# --------------------------------------------------------------------------
def features(X, omega):
    """Phi (n x 2m): row i = [cos 2 pi omega_k^T x_i (k<m), sin 2 pi omega_k^T x_i (k<m)].

    PAPER.md:318-320 (sigma_c(v) = exp(2 pi c i omega^T v) ...) with the
    real part kept as in the efficient estimator of PAPER.md:924-928
    (A3): exp(2 pi i w^T x_i) exp(-2 pi i w^T x_j) summed with the
    imaginary part dropped is cos(a_i) cos(a_j) + sin(a_i) sin(a_j).
    """
    theta = 2.0 * math.pi * (np.asarray(X, np.float64) @ np.asarray(omega, np.float64).T)
    return np.concatenate([np.cos(theta), np.sin(theta)], axis=1)


def estimator(z, omega, eps, c_r):
    """The paper's RF estimate of W(v, w) for z = n_v - n_w.

    W^(v, w) = (1/m) sum_i cos(2 pi omega_i^T z) tau(omega_i) / p(omega_i).
    """
    m = np.asarray(omega).shape[0]
    ang = 2.0 * math.pi * (np.asarray(z, np.float64) @ np.asarray(omega, np.float64).T)
    return np.cos(ang) @ (tau(omega, eps) / proposal_pdf(omega, c_r)) / m


# --------------------------------------------------------------------------
# a4, a6  sums over points
# --------------------------------------------------------------------------
def _chunk_sum(fn, n, chunk, init):
    """sum_{chunks in point order} fn(start, stop).  Chunk terms may be
    evaluated by a thread pool (numpy releases the GIL); they are added in
    chunk order, so the result does not depend on the thread count."""
    starts = list(range(0, n, chunk))
    workers = min(len(starts), os.cpu_count() or 1, 8)
    total = init
    if workers <= 1:
        for s in starts:
            total = total + fn(s, min(s + chunk, n))
        return total
    # One BLAS thread per worker: the pool already occupies the cores.
    with threadpoolctl.threadpool_limits(1), \
            concurrent.futures.ThreadPoolExecutor(max_workers=workers) as ex:
        for term in ex.map(lambda s: fn(s, min(s + chunk, n)), starts):
            total = total + term
    return total


def gram(X, omega, chunk=CHUNK):
    """G = Phi^T Phi (2m x 2m): B^T A of PAPER.md:337, 355 without D."""
    X = np.asarray(X)
    r = 2 * np.asarray(omega).shape[0]

    def term(s, e):
        P = features(X[s:e], omega)
        return P.T @ P
    return _chunk_sum(term, X.shape[0], chunk, np.zeros((r, r)))


def project(X, omega, F, chunk=CHUNK):
    """S = Phi^T F (2m x d): the first bracket B^T x of Eq. 13."""
    X = np.asarray(X)
    F = np.asarray(F, np.float64).reshape(X.shape[0], -1)
    r = 2 * np.asarray(omega).shape[0]

    def term(s, e):
        return features(X[s:e], omega).T @ F[s:e]
    return _chunk_sum(term, X.shape[0], chunk, np.zeros((r, F.shape[1])))


# --------------------------------------------------------------------------
# a5  core
# --------------------------------------------------------------------------
def phi1_lam(M, lam):
    """lam * phi1(lam M) = [exp(lam M) - I] M^{-1}, continuous at singular M.

    PAPER.md:333-339 (exp(L A B^T) = I + A [exp(L B^T A) - I](B^T A)^{-1} B^T)
    with the inverse removed by the series identity (A5;
    SPEC.md:408-416): the top-right block of
    expm([[lam M, lam I], [0, 0]]) is lam * phi1(lam M).
    """
    M = np.asarray(M, np.float64)
    r = M.shape[0]
    aug = np.zeros((2 * r, 2 * r))
    aug[:r, :r] = lam * M
    aug[:r, r:] = lam * np.eye(r)
    return scipy.linalg.expm(aug)[:r, r:]


def core(G, nu, lam):
    """C^ = D * lam * phi1(lam G D), D = diag(nu, nu) (2m x 2m).

    The middle factor [exp(L B^T A) - I](B^T A)^{-1} of Eq. 13
     with A = Phi D, B = Phi, so B^T A = G D, and the left
    factor A = Phi D contributing the leading D.
    """
    d = np.concatenate([nu, nu]).astype(np.float64)
    return d[:, None] * phi1_lam(G * d[None, :], lam)


# --------------------------------------------------------------------------
# NEXT-3  spectrum
# --------------------------------------------------------------------------
def spectrum(G, nu, lam, n, k):
    """The k smallest eigenvalues of K = exp(lam W~), W~ = Phi D Phi^T (N x N).

    PAPER.md:609 (classification "using the eigenvectors of the kernel
    matrix ... the k smallest eigenvalues"; low-rank route "as described in
    [nakatsukasa2019lowrank]"): the nonzero eigenvalues of
    A B^T = Phi D Phi^T are those of the 2m x 2m matrix B^T A = G D; each maps
    through exp(lam .), and the N - 2m null directions give eigenvalue 1.
    Reading (A19): for N < 2m, G D has 2m - N exact zero eigenvalues
    beyond W~'s N; the 2m - N of smallest modulus are dropped.
    """
    G = np.asarray(G, np.float64)
    r = G.shape[0]
    d = np.concatenate([nu, nu]).astype(np.float64)
    mu = np.linalg.eigvals(G * d[None, :])
    scale = max(1.0, float(np.abs(mu).max()))
    if np.abs(mu.imag).max() > 1e-8 * scale:
        raise ValueError("G D has non-real eigenvalues")
    mu = mu.real
    if n < r:
        mu = mu[np.argsort(np.abs(mu))[r - n:]]
    vals = np.exp(lam * mu)
    ones = np.ones(min(max(n - r, 0), k))
    return np.sort(np.concatenate([vals, ones]))[:k]


# --------------------------------------------------------------------------
# NEXT-1  Wasserstein barycenter (Alg. 1)
# --------------------------------------------------------------------------
BARY_CLAMP = 1e-30  # denominator clamp, SPEC.md:559 (A20)


def barycenter(apply_k, mus, area, alpha, max_iter, tol=0.0):
    """Entropic Wasserstein barycenter, Appendix D Algorithm 1
    (lines 1036-1051), with the readings of SPEC.md:559, 628-629 (DESIGN.md
    A20): mu reset to all-ones at each outer iteration; both denominators
    (FM_K(a v^i) and d^i) clamped at 1e-30, d^i before its power; stop after
    max_iter or when ||mu_new - mu_old||_1 < tol; output normalised so
    <a, mu> = 1.

    apply_k(X) applies the kernel FM_K to the columns of X (N x k).
    mus: k x N input distributions; area: N; alpha: k.
    Returns (mu, iterations run).
    """
    mus = np.asarray(mus, np.float64)
    k, N = mus.shape
    a = np.asarray(area, np.float64)
    al = np.asarray(alpha, np.float64)
    v = np.ones((N, k))
    mu = np.ones(N)
    it = 0
    for it in range(1, max_iter + 1):
        mu_old = mu
        # 1. w^i <- mu^i / FM_K(a * v^i)
        w = mus.T / np.maximum(apply_k(a[:, None] * v), BARY_CLAMP)
        # 2. d^i <- v^i * FM_K(a * w^i)  (the denominator of step 4 and the
        #    base of step 3's power; the random-feature kernel can map positive
        #    vectors to non-positive ones, so it is clamped too)
        dd = np.maximum(v * apply_k(a[:, None] * w), BARY_CLAMP)
        # 3. mu <- prod_i (d^i)^alpha_i   (mu reset to ones first)
        mu = np.prod(dd ** al[None, :], axis=1)
        # 4. v^i <- v^i * mu / d^i
        v = v * mu[:, None] / dd
        if not (np.isfinite(mu).all() and np.isfinite(v).all()):
            raise FloatingPointError("barycenter: non-finite iterate at iteration %d" % it)
        if tol > 0 and np.abs(mu - mu_old).sum() < tol:
            break
    return mu / float(a @ mu), it


# --------------------------------------------------------------------------
# plan + apply
# --------------------------------------------------------------------------
class Plan:
    """Pre-processing state ("pre-processing time linear in N
    and cubic in m"): omega, nu, G, C^ for one point cloud."""

    def __init__(self, X, eps, lam, m, seed, R=DEFAULT_R, c_r=None):
        self.X = np.asarray(X, np.float32)
        self.eps, self.lam, self.m, self.seed, self.R = eps, lam, m, seed, R
        self.c_r = l1_ball_mass(R) if c_r is None else c_r
        self.omega, self.attempts = frequencies(seed, m, R)
        self.nu = importance_weights(self.omega, eps, self.c_r)
        self.G = gram(self.X, self.omega)
        self.C = core(self.G, self.nu, lam)

    def reparam(self, eps, lam):
        """New (eps, lambda) on the stored G: G =
        B^T A depends on the points and omega only, eps enters
        through tau in nu, lambda through the core."""
        self.eps, self.lam = eps, lam
        self.nu = importance_weights(self.omega, eps, self.c_r)
        self.C = core(self.G, self.nu, lam)
        return self

    def spectrum(self, k):
        """k smallest eigenvalues of exp(lam W~) (NEXT-3; see ``spectrum``)."""
        return spectrum(self.G, self.nu, self.lam, self.X.shape[0], k)

    def barycenter(self, mus, area, alpha, max_iter, tol=0.0):
        """Alg. 1 with FM_K = this integrator (NEXT-1; see ``barycenter``)."""
        return barycenter(lambda X: self.apply(X)["out"], mus, area, alpha, max_iter, tol)

    def apply(self, F, rows=None):
        """Inference (Eq. 13, bracket order).

        Returns dict S, Y, out (out restricted to ``rows`` if given; every
        row still enters S).
        """
        F = np.asarray(F, np.float64).reshape(self.X.shape[0], -1)
        S = project(self.X, self.omega, F)
        Y = self.C @ S
        if rows is None:
            out = np.empty_like(F)
            for s in range(0, F.shape[0], CHUNK):
                out[s:s + CHUNK] = F[s:s + CHUNK] + features(
                    self.X[s:s + CHUNK], self.omega) @ Y
        else:
            rows = np.asarray(rows)
            out = F[rows] + features(self.X[rows], self.omega) @ Y
        return {"S": S, "Y": Y, "out": out}


def integrate(X, F, eps, lam, m, seed, R=DEFAULT_R):
    """One GFI with RFD: plan then apply.  Returns the plan and the results."""
    plan = Plan(X, eps, lam, m, seed, R)
    res = plan.apply(F)
    return plan, res
