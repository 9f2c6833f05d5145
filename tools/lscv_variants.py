"""A/B of the LSCV_h (d = 1) software-exp column masks on the C2 workload (GPU; one subprocess per
variant, KDE_DEBUG_LSCVh_SW): pair-kernel time of the 1024 candidates and parity against the C2
golden (stored oracle values; this tool never runs the oracle).

  python tools/lscv_variants.py [variants...]      (0 = default quarter mask, clamp-only exp)"""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, sys, time
sys.path.insert(0, os.environ["ROOT"])
import numpy as np, torch, datagen, paper_1505_01998_b200 as kb
ctx = kb.Context(profiling=True)
D = int(os.environ.get("LSCV_D", "1"))
if D == 1:
    X = datagen.config_data("C2"); Xd = kb.to_device(X); n = X.shape[1]
    h0 = (4.0 / (3.0 * n)) ** 0.2
    grid = np.linspace(h0 / 4, 4 * h0, 1024)
else:   # the F1 workload (tools/bench_configs.py F1)
    X = datagen.config_data("C5", n=65536)[:D]; Xd = kb.to_device(X); n = X.shape[1]
    grid = np.linspace(0.05, 1.5, 1024)
best = None
for _ in range(4):
    g = ctx.lscv_h_scores(Xd, grid)
    ms = ctx.last_profile()["pair_ms"]
    best = ms if best is None else min(best, ms)
err = None
if D == 1:
    gd = json.load(open(os.path.join(os.environ["ROOT"], "tests", "golden", "C2_lscv_h.json")))
    gs = ctx.lscv_h_scores(Xd, gd["h"])
    err = float(np.max(np.abs(gs - np.array(gd["g"])) / np.abs(gd["g"])))
print(json.dumps({"variant": int(os.environ.get("KDE_DEBUG_LSCVh_SW", "0")), "d": D, "pair_ms": best,
                  "evals_per_s": 2198989701120.0 / (best / 1e3), "max_rel_err_vs_golden": err}))
'''
for v in (sys.argv[1:] or ["0", "1", "2", "3", "4"]):
    env = dict(os.environ, KDE_DEBUG_LSCVh_SW=v, ROOT=ROOT)
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
    print(out.stdout.strip() or out.stderr[-500:], flush=True)
