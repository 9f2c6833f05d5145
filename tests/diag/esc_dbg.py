import sys, os, math, json
sys.path.insert(0, os.getcwd())
import numpy as np, datagen, oracle, paper_1505_01998_b200 as kb
ctx = kb.Context(profiling=True)
X = datagen.sample_mixture("skewed", 131109, 7)
Xd = kb.to_device(X)
s2p = math.sqrt(2 * math.pi)
for r, g in [(8, 0.2), (6, 0.2), (8, 0.05)]:
    ref = oracle.psi_pairsum(X[0], r, g, threads=len(os.sched_getaffinity(0)))
    out = {"r": r, "g": g, "oracle_S": ref}
    for mode in (-1, 0, 1):
        ctx.set_precision(mode)
        S = kb.fixed_value(ctx.raw_sums({4: kb.SUM_PSI4, 6: kb.SUM_PSI6, 8: kb.SUM_PSI8}[r], Xd, [g])[0]) / s2p
        out[f"mode{mode}"] = (S, ctx.last_fp64_passes(), ctx.last_psi_kappa())
        os.environ["KDE_DEBUG_PSI_NOSKIP"] = "1"
        S2 = kb.fixed_value(ctx.raw_sums({4: kb.SUM_PSI4, 6: kb.SUM_PSI6, 8: kb.SUM_PSI8}[r], Xd, [g])[0]) / s2p
        del os.environ["KDE_DEBUG_PSI_NOSKIP"]
        out[f"mode{mode}_noskip"] = S2
    print(json.dumps(out), flush=True)
# psi_r (the public call) on the same data, in every mode
for mode in (-1, 0, 1):
    ctx.set_precision(mode)
    for r, g in [(8, 0.2), (6, 0.2)]:
        v = ctx.psi_r(Xd, r, [g])[0]
        ref = oracle.psi_r(X[0], r, g, threads=len(os.sched_getaffinity(0)))
        print(json.dumps({"psi_r": True, "mode": mode, "r": r, "g": g, "got": v, "ref": ref, "passes": ctx.last_fp64_passes()}), flush=True)
