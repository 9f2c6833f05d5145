"""Randomised check of the bounded far-tile skip on the GPU: for random sample shapes,
sizes and bandwidths, the default pass (bounded skip) against the same pass without any skip.
  Psi_r: |S_bounded - S_noskip| <= 1e-9 |2 S + n He_r(0)|   (fp32 terms, psi mode -1)
  LSCV:  0 <= S_noskip - S_bounded <= n(n-1)/2 2^-theta (S1), 2^-2theta (S2)
Prints one line per case and the worst ratio (dropped / bound).  usage: skip_fuzz.py [cases] [seed]"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import datagen  # noqa: E402
import paper_1505_01998_b200 as kb  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
ctx = kb.Context(profiling=True)
ctx.set_precision(-1)


def sample(kind, n, d):
    if kind == "normal":
        return rng.normal(size=(d, n))
    if kind == "mixture":
        c = rng.integers(0, 3, n)
        return rng.normal(size=(d, n)) * (0.2 + c * 0.3) + c * 2.0
    if kind == "spikes":
        return rng.integers(0, 8, (1, n)) * 3.0 + rng.normal(0, 0.02, (d, n))
    if kind == "t3":
        return rng.standard_t(3, size=(d, n))
    return rng.uniform(-1, 1, size=(d, n))


def noskip(fn):
    os.environ["KDE_DEBUG_PSI_NOSKIP"] = "1"
    os.environ["KDE_DEBUG_LSCV_NOSKIP"] = "1"
    try:
        return fn()
    finally:
        del os.environ["KDE_DEBUG_PSI_NOSKIP"], os.environ["KDE_DEBUG_LSCV_NOSKIP"]


worst = {"psi": 0.0, "lscv": 0.0}
skipped = {"psi": [], "lscv": []}
for c in range(cases):
    kind = ["normal", "mixture", "spikes", "t3", "uniform"][rng.integers(0, 5)]
    if c % 2 == 0:   # Psi
        n = int(np.exp(rng.uniform(np.log(3000), np.log(300000))))
        x = sample(kind, n, 1)
        sd = float(np.std(x))
        r = [4, 6, 8][rng.integers(0, 3)]
        g = sd * float(np.exp(rng.uniform(np.log(0.003), np.log(2.0))))
        X = kb.to_device(x)
        a = ctx.raw_sums(r, X, [g])
        ev = ctx.last_profile()["pair_evals"]
        b = noskip(lambda: ctx.raw_sums(r, X, [g]))
        full = ctx.last_profile()["pair_evals"]
        Sa, Sb = kb.fixed_value(a[0]), kb.fixed_value(b[0])
        he0 = {4: 3.0, 6: -15.0, 8: 105.0}[r]
        ratio = abs(Sa - Sb) / (1e-9 * abs(2 * Sb + n * he0))
        worst["psi"] = max(worst["psi"], ratio)
        skipped["psi"].append(1 - ev / full)
        print("psi %-7s n=%6d r=%d g/sd=%.4f tau=%.3f skipped=%.3f dropped/bound=%.2e"
              % (kind, n, r, g / sd, kb.psi_skip_gap(r, g, float(np.var(x, ddof=1))), 1 - ev / full, ratio))
    else:            # LSCV_h (d = 1..3) or LSCV_H (d = 2, 4)
        d = int(rng.integers(1, 5))
        n = int(np.exp(rng.uniform(np.log(2000), np.log(40000))))
        x = sample(kind, n, d)
        X = kb.to_device(x)
        theta = kb.lscv_skip_theta(n)
        if d in (2, 4) and rng.uniform() < 0.5:
            C = np.cov(x)
            cands = np.concatenate([datagen.vech(C * s) for s in np.exp(rng.uniform(np.log(1e-3), np.log(0.5), 4))])
            kind_s, nc = kb.SUM_LSCV_H, 4
        else:
            cands = np.exp(rng.uniform(np.log(0.005), np.log(1.5), 12))
            kind_s, nc = kb.SUM_LSCV_h, 12
        a = ctx.raw_sums(kind_s, X, cands)
        ev = ctx.last_profile()["pair_evals"]
        b = noskip(lambda: ctx.raw_sums(kind_s, X, cands))
        full = ctx.last_profile()["pair_evals"]
        pairs = n * (n - 1) / 2
        ratio = 0.0
        for k in range(nc):
            for j, p in ((0, 1.0), (1, 2.0)):
                dS = kb.fixed_value(b[2 * k + j]) - kb.fixed_value(a[2 * k + j])
                assert dS >= 0.0, (c, k, j, dS)
                ratio = max(ratio, dS / (pairs * 2.0 ** (-p * theta)))
        worst["lscv"] = max(worst["lscv"], ratio)
        skipped["lscv"].append(1 - ev / full)
        print("lscv%s %-7s n=%6d d=%d theta=%.1f skipped=%.3f dropped/bound=%.2e"
              % ("H" if kind_s == kb.SUM_LSCV_H else "h", kind, n, d, theta, 1 - ev / full, ratio))
print("cases %d worst dropped/bound: psi %.3e lscv %.3e; mean skipped fraction psi %.3f lscv %.3f"
      % (cases, worst["psi"], worst["lscv"], np.mean(skipped["psi"]), np.mean(skipped["lscv"])))
assert worst["psi"] <= 1.0 and worst["lscv"] <= 1.0001
