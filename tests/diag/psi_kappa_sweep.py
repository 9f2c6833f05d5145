"""Library-only sweep of the Psi cancellation estimate kappa (GPU diagnostic, no oracle): which
(data, n, r, g) exceed kPsiKappaMax, and kappa at the C4 / C4b PLUGIN workloads."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import datagen
import paper_1505_01998_b200 as kb

ctx = kb.Context()
ctx.set_precision(-1)
for name, n, seed in [("skewed", 131109, 7), ("skewed", 1 << 20, 4), ("bimodal", 131109, 2), ("N01", 131109, 1),
                      ("kurtotic", 1 << 20, 14), ("skewed", 300001, 8)]:
    X = datagen.sample_mixture(name, n, seed)
    Xd = kb.to_device(X)
    for r in (4, 6, 8):
        for g in (0.05, 0.1, 0.2, 0.3, 0.5, 1.0, 2.0):
            kind = {4: kb.SUM_PSI4, 6: kb.SUM_PSI6, 8: kb.SUM_PSI8}[r]
            ctx.raw_sums(kind, Xd, [g])
            print(json.dumps({"data": name, "n": n, "seed": seed, "r": r, "g": g, "kappa": ctx.last_psi_kappa()}), flush=True)
for name, X in [("C4", datagen.config_data("C4")), ("C4b", datagen.sample_mixture("kurtotic", 1 << 20, 14))]:
    h, tr = ctx.plugin_h(kb.to_device(X))
    print(json.dumps({"plugin": name, "kappa_max": ctx.last_psi_kappa(), "g1": tr["g1"], "g2": tr["g2"]}), flush=True)
