"""Extended seeded fuzz (GPU vs oracle), the same checks as tests/test_gpu_fuzz.py on many more
random (n, d, bandwidth scale) cases; prints the worst relative errors per family and every case
over the 1e-5 contract.  Usage: python tests/diag/fuzz_wide.py [cases] [seed] [dmax] [nmax]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1505_01998_b200 as kb  # noqa: E402


def _data(n, d, seed):
    r = np.random.default_rng(seed)
    A = r.normal(size=(d, d)) / np.sqrt(d) + np.eye(d)
    X = A @ r.standard_t(5, size=(d, n))
    return X + r.normal(size=(d, 1)) * 3


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
    dmax = int(sys.argv[3]) if len(sys.argv) > 3 else 6      # d drawn from 1..dmax
    nmax = int(sys.argv[4]) if len(sys.argv) > 4 else 4000
    ctx = kb.Context()
    worst = {"psi": 0.0, "lscv_h": 0.0, "lscv_H": 0.0}
    worst_pt = {"lscv_h": 0.0, "lscv_H": 0.0}   # pointwise |got - ref| / |ref| (north_star criterion)
    near_zero = []
    bad = []
    for c in range(cases):
        n = int(rng.integers(2, nmax))
        d = int(rng.integers(1, dmax + 1))
        scale = float(10 ** rng.uniform(-1.3, 0.3))
        X = _data(n, d, 1000 + c)
        x1 = np.ascontiguousarray(X[:1])
        g = scale * max(np.std(x1), 1e-3)
        for r in (4, 6, 8):
            got = ctx.psi_r(kb.to_device(x1), r, [g])[0]
            ref = oracle.psi_r(x1[0], r, g)
            e = abs(got - ref) / abs(ref)
            worst["psi"] = max(worst["psi"], e)
            if e > 1e-5:
                bad.append(("psi", n, d, r, scale, e))
        _, S = oracle.mean_cov(X)
        if n < 3 or np.linalg.cond(S) > 1e8:
            continue
        Xd = kb.to_device(X)
        hs = np.array([0.5, 1.0, 2.0]) * scale
        for fam, got, ref in (("lscv_h", ctx.lscv_h_scores(Xd, hs), oracle.lscv_h_scores(X, hs)),
                              ("lscv_H", ctx.lscv_H_scores(Xd, [datagen.vech(h * h * S) for h in hs]),
                               [oracle.lscv_H_score(X, datagen.vech(h * h * S)) for h in hs])):
            # Two measures.  Pointwise relative error (the north_star 1e-5 criterion), reported
            # in full; and relative to the curve's scale, because an objective can cross zero
            # between grid points (case 28 of seed 7: g = 7.4e-8 between 3.0e-3 and -9.0e-5),
            # where the pointwise ratio measures the cancellation of g itself, not the kernel.
            got, ref = np.asarray(got), np.asarray(ref)
            pt = np.abs(got - ref) / np.abs(ref)
            e = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
            worst[fam] = max(worst[fam], e)
            worst_pt[fam] = max(worst_pt[fam], float(pt.max()))
            for k in range(len(hs)):
                if pt[k] > 1e-5:
                    zc = abs(ref[k]) < 1e-3 * np.max(np.abs(ref))
                    (near_zero if zc else bad).append((fam, n, d, scale, float(hs[k]), float(ref[k]), float(pt[k])))
            if e > 1e-5:
                bad.append((fam, n, d, scale, "curve-scale", e))
    print("cases", cases, "worst (curve scale)", worst, "worst (pointwise)", worst_pt)
    for z in near_zero:
        print("pointwise > 1e-5 at |g| < 1e-3 max|g| (zero crossing):", z)
    for b in bad:
        print("OVER 1e-5:", b)


if __name__ == "__main__":
    main()
