"""Diagnose one wide-fuzz LSCV case (GPU vs oracle): raw sums S1 = sum e^{-q/4}, S2 = sum e^{-q/2}
of both LSCV families, their relative errors, the objective's cancellation (A + B) / |g|, and the
effect of the far-tile skip.  python tests/diag/lscv_case.py [n d seed_of_fuzz]"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import datagen, oracle
import paper_1505_01998_b200 as kb
sys.path.insert(0, os.path.join(os.getcwd(), "tests", "diag"))
from fuzz_wide import _data

n_t, d_t, seed = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (1671, 3, 7)
rng = np.random.default_rng(seed)
for c in range(5000):
    n = int(rng.integers(2, 4000)); d = int(rng.integers(1, 7)); scale = float(10 ** rng.uniform(-1.3, 0.3))
    if n == n_t and d == d_t:
        break
X = _data(n, d, 1000 + c)
_, S = oracle.mean_cov(X)
ctx = kb.Context()


def val(f):
    k, S = f.key()
    return float(k) * 2.0 ** -S


Xd = kb.to_device(X)
hs = np.array([0.5, 1.0, 2.0]) * scale
print("case", c, "n", n, "d", d, "scale", scale, "max|x'|/h", float(np.max(np.abs(np.linalg.solve(np.linalg.cholesky(S), X - X.mean(1, keepdims=True))))) / hs[0])
for h in hs:
    H = datagen.vech(h * h * S)
    gref, (A1, B1) = oracle.lscv_H_score(X, H, parts=True)
    g = ctx.lscv_H_scores(Xd, [H])[0]
    gh = ctx.lscv_h_scores(Xd, [h])[0]
    grefh, parts = oracle.lscv_h_scores(X, [h], parts=True)
    s = ctx.raw_sums(kb.SUM_LSCV_H, Xd, H)
    sh = ctx.raw_sums(kb.SUM_LSCV_h, Xd, [h])
    det = np.linalg.det(h * h * S)
    c4 = (4 * np.pi) ** (-d / 2) * det ** -0.5; c2 = (2 * np.pi) ** (-d / 2) * det ** -0.5
    S1r, S2r = A1 / c4, B1 / c2
    S1, S2 = val(s[0]), val(s[1])
    S1h, S2h = val(sh[0]), val(sh[1])
    kap = (2 * A1 / n**2 + 4 * B1 / n**2) / abs(gref)
    os.environ["KDE_DEBUG_LSCV_NOSKIP"] = "1"
    gns = ctx.lscv_H_scores(Xd, [H])[0]
    del os.environ["KDE_DEBUG_LSCV_NOSKIP"]
    print(f"h {h:.4g} g_ref {gref:.6e} kappa' {kap:.1f} | H: rel g {abs(g-gref)/abs(gref):.2e} S1 {abs(S1-S1r)/S1r:.2e} "
          f"S2 {abs(S2-S2r)/S2r:.2e} noskip-equal {gns == g} | h: rel g {abs(gh-grefh[0])/abs(grefh[0]):.2e} "
          f"S1 {abs(S1h-S1r)/S1r:.2e} S2 {abs(S2h-S2r)/S2r:.2e}")
