"""Psi accuracy probe (GPU): raw pair sums vs the fp64 oracle on hard cases, and the C4 trace vs its golden (see profiles/r01_psi_accuracy.md)."""
import json, math, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import datagen, oracle, paper_1505_01998_b200 as kb
ctx = kb.Context()
s2p = math.sqrt(2 * math.pi)
cases = [(131109, 6, 0.2), (131109, 4, 0.1), (131109, 6, 0.05), (40000, 6, 0.02), (300000, 6, 0.2), (300000, 4, 0.11)]
xbig = datagen.sample_mixture("skewed", 300000, 7)
out = []
for n, r, g in cases:
    x = xbig[:, :n]
    cache = f"/tmp/psiref_{n}_{r}_{g}.npy"
    if os.path.exists(cache):
        ref = float(np.load(cache))
    else:
        ref = oracle.psi_pairsum(x[0], r, g, threads=len(os.sched_getaffinity(0)))
        np.save(cache, ref)
    kind = {4: kb.SUM_PSI4, 6: kb.SUM_PSI6, 8: kb.SUM_PSI8}[r]
    got = kb.fixed_value(ctx.raw_sums(kind, kb.to_device(x), [g])[0]) / s2p
    out.append((n, r, g, (got - ref) / abs(ref)))
gold = json.load(open("tests/golden/C4_plugin.json"))["trace"] if os.path.exists("tests/golden/C4_plugin.json") else None
if gold:
    h, tr = ctx.plugin_h(kb.to_device(datagen.config_data("C4")))
    out.append(("C4", "psi6", (tr["psi6"] - gold["psi6"]) / abs(gold["psi6"])))
    out.append(("C4", "psi4", (tr["psi4"] - gold["psi4"]) / abs(gold["psi4"])))
for o in out:
    print(o)
