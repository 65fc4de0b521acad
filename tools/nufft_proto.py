import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
from oracle import rfd as O
from workloads import configs as C

def es(z, beta):
    out = np.zeros_like(z)
    msk = np.abs(z) < 1
    out[msk] = np.exp(beta * (np.sqrt(1 - z[msk] ** 2) - 1))
    return out

def phihat(s, alpha, beta, nq=200):
    z, wq = np.polynomial.legendre.leggauss(nq)
    psi = es(z, beta)
    return alpha * (np.cos(np.outer(s, alpha * z)) @ (wq * psi))

F32 = False
def nufft_gram(X, omega, w=8, hfac=1.5, betaf=2.30):
    beta = betaf * w
    lo, hi = X.min(0), X.max(0)
    c = 0.5 * (lo + hi)
    Y = X - c
    Xh = 0.5 * (hi - lo)
    S = 2 * np.pi * 2 * np.abs(omega).max(0)          # rad per unit
    h = hfac / S
    if F32:  # h = q * 2^-e, q < 16
        e = np.floor(np.log2(h)) - 3
        h = np.floor(h / 2.0**e) * 2.0**e
        Y = Y.astype(np.float32).astype(np.float64)
    alpha = w * h / 2
    # grid nodes: l = -L..L with L covering Xh + alpha
    L = np.ceil((Xh + alpha) / h).astype(int) + 1
    n = 2 * L + 1
    b = np.zeros(tuple(n))
    # spreading: each point to nodes within alpha
    idx = []
    vals = []
    for a in range(3):
        l0 = np.ceil((Y[:, a] - alpha[a]) / h[a]).astype(int)   # first node >= x - alpha
        ls = l0[:, None] + np.arange(w + 1)[None, :]
        if F32:
            z = ((np.float32(1) * (ls * h[a]).astype(np.float32) - Y[:, a:a+1].astype(np.float32)) * np.float32(1 / alpha[a])).astype(np.float32)
            v = np.zeros_like(z); mk = np.abs(z) < 1
            v[mk] = np.exp(np.float32(beta) * (np.sqrt(np.float32(1) - z[mk] * z[mk]) - np.float32(1)))
            vals.append(v.astype(np.float64))
        else:
            z = (ls * h[a] - Y[:, a:a+1]) / alpha[a]
            vals.append(es(z, beta))
        idx.append(ls + L[a])
    for i in range(w + 1):
        for j in range(w + 1):
            vxy = vals[0][:, i] * vals[1][:, j]
            for k in range(w + 1):
                if F32:
                    pr = np.rint((vxy.astype(np.float32) * np.float32(2**22)).astype(np.float32) * vals[2][:, k].astype(np.float32)).astype(np.float64) / 2**22
                else:
                    pr = vxy * vals[2][:, k]
                np.add.at(b, (idx[0][:, i], idx[1][:, j], idx[2][:, k]), pr)
    # grid nodes
    g = np.stack(np.meshgrid(*[(np.arange(n[a]) - L[a]) * h[a] for a in range(3)], indexing="ij"), -1).reshape(-1, 3)
    bw = b.reshape(-1)
    keep = bw > 0
    g, bw = g[keep], bw[keep]
    th = 2 * np.pi * g @ omega.T                       # (ng, m)
    cs, sn = np.cos(th), np.sin(th)
    cc = (cs * bw[:, None]).T @ cs
    ss = (sn * bw[:, None]).T @ sn
    sc = (sn * bw[:, None]).T @ cs   # sum sin_j cos_k
    cs_ = (cs * bw[:, None]).T @ sn  # sum cos_j sin_k
    Pp_re, Pp_im = cc - ss, sc + cs_
    Pm_re, Pm_im = cc + ss, sc - cs_
    m = omega.shape[0]
    sp = 2 * np.pi * (omega[:, None, :] + omega[None, :, :])
    sm = 2 * np.pi * (omega[:, None, :] - omega[None, :, :])
    def deconv(s):
        f = np.ones(s.shape[:2])
        for a in range(3):
            f *= phihat(s[..., a].reshape(-1), alpha[a], beta).reshape(s.shape[:2]) / h[a]
        return f
    dp, dm = deconv(sp), deconv(sm)
    Pp = (Pp_re + 1j * Pp_im) / dp
    Pm = (Pm_re + 1j * Pm_im) / dm
    Gcc = 0.5 * (Pm.real + Pp.real)
    Gss = 0.5 * (Pm.real - Pp.real)
    Gcs = 0.5 * (Pp.imag - Pm.imag)
    Gsc = 0.5 * (Pp.imag + Pm.imag)
    G = np.zeros((2 * m, 2 * m))
    G[:m, :m] = Gcc; G[m:, m:] = Gss; G[:m, m:] = Gcs; G[m:, :m] = Gsc
    return G, c, n, g.shape[0], np.abs(dp).min() / dp.max()

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
npts = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
m = int(sys.argv[3]) if len(sys.argv) > 3 else 256
params, X, F = C.make_config(cfg, n=npts)
X = np.asarray(X, dtype=np.float64)
print(params)
omega = np.asarray(O.frequencies(params["seed"], m)[0])
lo, hi = X.min(0), X.max(0); c = 0.5 * (lo + hi)
t = time.time(); Gd = O.gram(X - c, omega); print("direct", time.time() - t)
F32 = len(sys.argv) > 5
for w in [int(a) for a in (sys.argv[4].split(",") if len(sys.argv) > 4 else ["6", "7", "8"])]:
    for hf in [1.5, 1.2]:
        t = time.time(); Gn, _, n, ng, dr = nufft_gram(X, omega, w=w, hfac=hf)
        err = np.abs(Gn - Gd).max() / np.abs(Gd).max()
        print(f"w={w} hfac={hf} grid={tuple(n)} nodes={ng} minratio={dr:.3g} normwise={err:.3g} t={time.time()-t:.1f}s")
