"""Psi_6 pair-kernel throughput vs n (tile size switches at n = 64 * 2048)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_1505_01998_b200 as kb
ctx = kb.Context(profiling=True)
for n in (20000, 60000, 100000, 131071, 131072, 262144):
    x = kb.to_device(datagen.sample_mixture("skewed", n, 3))
    best = None
    for _ in range(3):
        ctx.psi_r(x, 6, [0.2])
        p = ctx.last_profile()
        best = p if best is None or p["pair_ms"] < best["pair_ms"] else best
    ev = best["pair_evals"]
    print(json.dumps({"n": n, "pair_ms": best["pair_ms"], "evals_per_s": ev / best["pair_ms"] * 1e3,
                      "frac_mufu": ev / best["pair_ms"] * 1e3 / 4.65312e12}), flush=True)
