"""Psi precision calibration (GPU diagnostic, calls the oracle): for each case the fp32-term pass's
error against the fp64 oracle (kde_set_precision -1), the library's cancellation estimate kappa,
and the automatic mode's result (fp64 re-run when kappa > kPsiKappaMax).  Output: one JSON per
line (profiles/r02_psi_kappa.jsonl).  python tests/diag/psi_kappa.py [--quick]"""
import json, math, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import datagen, oracle
import paper_1505_01998_b200 as kb

THREADS = len(os.sched_getaffinity(0))
s2p = math.sqrt(2 * math.pi)
ctx = kb.Context()
quick = "--quick" in sys.argv


def spiky(n, seed, k=12, w=0.01):
    # k tight clusters (sd w) on [0, 10]: heavy cancellation at the PLUGIN pilot bandwidths
    u = datagen.uniforms(seed, 0, n)
    z = datagen.normals(seed, n, n)
    return (np.floor(u * k) * (10.0 / k) + w * z)[None, :]


cases = []
xs = datagen.sample_mixture("skewed", 300000, 7)
for n, gs, rs in [(5000, [0.01, 0.05, 0.3], [4, 6, 8]), (40000, [0.005, 0.01, 0.02, 0.05, 0.1, 0.2], [4, 6, 8]),
                  (131109, [0.05, 0.1, 0.2], [4, 6])]:
    if quick and n > 40000:
        continue
    for g in gs:
        for r in rs:
            cases.append(("skewed7", xs[:, :n], r, g))
xn = datagen.sample_mixture("N01", 40000, 11)
for g in [0.003, 0.01, 0.05]:
    cases.append(("N01", xn, 6, g))
for n, w_ in [(20000, 0.01), (20000, 0.001)]:
    xk = spiky(n, 13, w=w_)
    for g in [0.002, 0.01, 0.05, 0.3]:
        cases.append((f"spiky{w_}", xk, 6, g))
        cases.append((f"spiky{w_}", xk, 4, g))

kind = {4: kb.SUM_PSI4, 6: kb.SUM_PSI6, 8: kb.SUM_PSI8}
for name, X, r, g in cases:
    n = X.shape[1]
    t0 = time.time()
    ref_S = oracle.psi_pairsum(X[0], r, g, threads=THREADS)
    he0 = {4: 3.0, 6: -15.0, 8: 105.0}[r]
    ref = (2 * ref_S + n * he0)
    Xd = kb.to_device(X)
    ctx.set_precision(-1)
    S32 = kb.fixed_value(ctx.raw_sums(kind[r], Xd, [g])[0]) / s2p
    kappa = ctx.last_psi_kappa()
    ctx.set_precision(0)
    Sa = kb.fixed_value(ctx.raw_sums(kind[r], Xd, [g])[0]) / s2p
    passes = ctx.last_fp64_passes()
    e32 = (2 * S32 + n * he0 - ref) / abs(ref)
    ea = (2 * Sa + n * he0 - ref) / abs(ref)
    print(json.dumps({"data": name, "n": n, "r": r, "g": g, "kappa": kappa, "err_fp32": e32,
                      "err_fp32_over_kappa": abs(e32) / kappa if kappa else None,
                      "auto_fp64_passes": passes, "err_auto": ea, "oracle_s": round(time.time() - t0, 2)}), flush=True)

# PLUGIN chain: the device-side gate
for name, X in [("C1", datagen.config_data("C1")), ("skewed7_40000", xs[:, :40000]),
                ("spiky0.01", spiky(20000, 13, w=0.01)), ("spiky0.001", spiky(20000, 13, w=0.001))]:
    ref = oracle.plugin(X[0], threads=THREADS)
    Xd = kb.to_device(X)
    out = {"data": name, "n": X.shape[1], "plugin": True}
    for mode in (-1, 0, 1):
        ctx.set_precision(mode)
        try:
            h, tr = ctx.plugin_h(Xd)
            out[f"mode{mode}"] = {"psi6_err": (tr["psi6"] - ref["psi6"]) / abs(ref["psi6"]),
                                  "psi4_err": (tr["psi4"] - ref["psi4"]) / abs(ref["psi4"]),
                                  "h_err": (h - ref["h"]) / ref["h"], "kappa": ctx.last_psi_kappa(),
                                  "fp64_passes": ctx.last_fp64_passes()}
        except kb.KDEError as e:
            out[f"mode{mode}"] = {"error": str(e)}
    ctx.set_precision(0)
    print(json.dumps(out), flush=True)
