import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, datagen, paper_1505_01998_b200 as kb
ctx = kb.Context()
def val(f):
    k, S = f.key(); return float(k) * 2.0 ** -S
for name in ("C2", "F1d2"):
    X = datagen.config_data("C2") if name == "C2" else datagen.sample_mixture("C3", 65536, 7)
    d, n = X.shape
    h0 = (4.0 / (3.0 * n)) ** 0.2 if d == 1 else None
    grid = np.linspace(h0 / 4, 4 * h0, 1024) if d == 1 else np.linspace(0.05, 0.8, 1024)
    g = ctx.lscv_h_scores(kb.to_device(X), grid)
    s = ctx.raw_sums(kb.SUM_LSCV_h, kb.to_device(X), grid)
    S = np.cov(X) if d > 1 else np.array([[np.var(X, ddof=1)]])
    det = np.linalg.det(S)
    kaps = []
    for k, h in enumerate(grid):
        S1, S2 = val(s[2 * k]), val(s[2 * k + 1])
        c4 = (4 * np.pi) ** (-d / 2) / np.sqrt(det); c2 = (2 * np.pi) ** (-d / 2) / np.sqrt(det)
        A = h ** -d * 2 * c4 * S1 / n**2; B = h ** -d * 4 * c2 * S2 / n**2
        kaps.append((A + B) / abs(g[k]))
    kaps = np.array(kaps)
    print(name, "kappa' max %.1f, count > 32: %d, > 16: %d, > 8: %d, argmax h %.4f g %.3e" % (kaps.max(), (kaps > 32).sum(), (kaps > 16).sum(), (kaps > 8).sum(), grid[kaps.argmax()], g[kaps.argmax()]))
