import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2302_00942_b200 import rfd
from oracle import rfd as orf
rfd.load_library()
rng = np.random.default_rng(11)
n = 4096
for shape in ("point", "line"):
    x = np.zeros((n, 3))
    if shape != "point":
        x[:, 0] = rng.uniform(-0.5, 0.5, n)
    x = (x + np.array([0.25, -1.0, 3.0])).astype(np.float32)
    ref = orf.Plan(x, 0.05, -0.4, 128, 6)
    Gs = {}
    for mode in ("0", "2"):
        os.environ["RFD_GRAM_SPREAD"] = mode
        pl = rfd.Plan(torch.from_numpy(x).cuda(), 0.05, -0.4, 128, 6)
        G = pl.export("gram"); C = pl.export("core")
        Gs[mode] = G
        eG = np.abs(G - ref.G).max() / np.abs(ref.G).max(); eC = np.abs(C - ref.C).max() / np.abs(ref.C).max()
        print(shape, mode, "nodes", pl.info()["gram_nodes"], "G %.2e C %.2e" % (eG, eC), "scaling", pl.info()["scaling"])
    d = np.abs(Gs["2"] - ref.G)
    i = np.unravel_index(d.argmax(), d.shape)
    print("  worst G entry", i, Gs["2"][i], ref.G[i], "diag max", np.abs(np.diag(ref.G)).max())
    w = np.linalg.eigvalsh(ref.G); print("  G eig top", w[-3:], "G_spread eig top", np.linalg.eigvalsh(Gs["2"])[-3:], "min", np.linalg.eigvalsh(Gs["2"])[:3])
