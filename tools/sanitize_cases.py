"""Small invocations of every kernel family, for compute-sanitizer (memcheck/racecheck/synccheck)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_1505_01998_b200 as kb  # noqa: E402

ctx = kb.Context()
x = kb.to_device(datagen.sample_mixture("skewed", 1500, 1))
print("plugin", ctx.plugin_h(x)[0])
print("psi8", ctx.psi_r(x, 8, [0.3]))
X = kb.to_device(datagen.sample_mixture("C3", 700, 2))
print("lscv_h", ctx.lscv_h_scores(X, np.linspace(0.1, 1, 5)))
print("lscv_H", ctx.lscv_H_scores(X, [[0.05, 0.01, 0.04], [0.2, -0.02, 0.1]]))
X5 = kb.to_device(np.random.default_rng(1).normal(size=(5, 300)))
print("lscv_H d5", ctx.lscv_H_scores(X5, [np.eye(5)[np.tril_indices(5)[::-1]].ravel() * 0 + datagen.vech(np.eye(5) * 0.3)]))
print("eval", ctx.evaluate(X, kb.to_device(datagen.sample_mixture("C3", 600, 3)), [0.05, 0.0, 0.05])[:3])
print("aqp", ctx.aqp_1d(x, 0.2, [-1.0], [1.0]))
print("materialized", ctx.lscv_h_scores_materialized(X, np.linspace(0.1, 1, 4), 4))
print("select H", ctx.select_bandwidth(kb.LSCV_H, X, max_iter=5)["objective"])
print("select H multistart", ctx.select_bandwidth(kb.LSCV_H, X, max_iter=8, nm_starts=3)["objective"])
print("select h refine", ctx.select_bandwidth(kb.LSCV_h, X, n_grid=20, refine_steps=2)["h"])
print("plugin host input", ctx.plugin_h(datagen.sample_mixture("skewed", 1500, 1))[0])
print("psi shards", [kb.fixed_value(f) for r in range(3) for f in ctx.raw_sums(kb.SUM_PSI6, x, [0.3], shard=(r, 3))])
print("select plugin", ctx.select_bandwidth(kb.PLUGIN, x)["h"])
print("lscv_H 300 candidates (two launches)", ctx.lscv_H_scores(X, np.tile([[0.05, 0.01, 0.04]], (300, 1)))[[0, 299]])
xs = kb.to_device(datagen.sample_mixture("skewed", 700, 3))
print("plugin x3 (graph capture + replay)", [ctx.plugin_h(xs)[0] for _ in range(3)])
ctx.set_precision(True)
print("fp64 psi + plugin", ctx.psi_r(x, 6, [0.3]), ctx.plugin_h(x)[0])
ctx.set_precision(False)
# round 2: LSCV far-tile skip on sorted data, fp64-term LSCV (prep64 + lscv64), the device Nelder-Mead
# loop (PDL launches, 4 rounds per condition), skipped-tile NM
Xb = kb.to_device(datagen.sample_mixture("bimodal", 3001, 4))
print("lscv_h skip", ctx.lscv_h_scores(Xb, [0.005, 0.01, 0.5]))
X3 = kb.to_device(datagen.sample_mixture("C5", 2100, 5)[:3])
print("lscv_H skip", ctx.lscv_H_scores(X3, [datagen.vech(np.eye(3) * 1e-4), datagen.vech(np.eye(3) * 0.05)]))
ctx.set_precision(1)
print("fp64 lscv", ctx.lscv_h_scores(X, [0.3]), ctx.lscv_H_scores(X3, [datagen.vech(np.eye(3) * 0.05)]))
ctx.set_precision(0)
print("select H device loop", ctx.select_bandwidth(kb.LSCV_H, X, max_iter=40)["objective"])
# round 2, second part: bounded far-tile skip (Psi tau from g/sigma, LSCV theta = log2 n + 30, per-candidate
# tile bound inside an LSCV_h batch) and multi-launch passes on two streams (24 h = 3 launches)
print("lscv_h two streams + per-candidate skip", ctx.lscv_h_scores(Xb, np.geomspace(0.003, 1.0, 24))[[0, 23]])
print("psi bounded skip", ctx.psi_r(x, 4, [0.02, 0.3]))
