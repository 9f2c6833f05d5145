"""Write the full-size golden values of the BASELINE.json configs with the fp64 oracle.

Calls only oracle/ (and datagen for the seeded inputs).  Each JSON file records the workload,
the oracle outputs and the PAPER.md passages they follow.  Run (CPU, all cores, ~1 h):

    python tests/golden/make_golden.py [C1] [C4] [C2] [C3] [C5] [C4b] [T2048] [C5small] [ESC] [F1] [F2]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle   # noqa: E402

THREADS = len(os.sched_getaffinity(0))


def dump(name, obj):
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(obj, f, indent=1)


def c1():
    x = datagen.config_data("C1")[0]
    t0 = time.time()
    tr = oracle.plugin(x)
    dump("C1_plugin.json", {
        "config": "C1", "workload": "PLUGIN, n=1000, N(0,1), datagen seed 1",
        "cite": "PAPER.md P:203-256 (Sec. 4.4.1 steps 1-8, Eq. 11-18), reading Z1 for Eq. 15/17",
        "trace": tr, "oracle_seconds": time.time() - t0, "threads": 1})


def c4():
    x = datagen.config_data("C4")[0]
    t0 = time.time()
    tr = oracle.plugin(x, threads=THREADS)
    dump("C4_plugin.json", {
        "config": "C4", "workload": "PLUGIN, n=2^20, Marron-Wand #2 skewed mixture, datagen seed 4",
        "cite": "PAPER.md P:203-256 (Sec. 4.4.1 steps 1-8, Eq. 11-18), reading Z1 for Eq. 15/17",
        "trace": tr, "oracle_seconds": time.time() - t0, "threads": THREADS})


def c2():
    X = datagen.config_data("C2")
    n = X.shape[1]
    grid = oracle.lscv_h_grid(n, 1, 1024, 4.0)
    t0 = time.time()
    coarse = list(range(0, 1024, 32)) + [1023]
    sc = oracle.lscv_h_scores(X, grid[coarse], threads=THREADS)
    k0 = coarse[int(np.argmin(sc))]
    fine = [k for k in range(max(0, k0 - 24), min(1024, k0 + 25)) if k not in coarse]
    sf = oracle.lscv_h_scores(X, grid[fine], threads=THREADS)
    idx = coarse + fine
    vals = list(sc) + list(sf)
    order = np.argsort(idx)
    idx = [int(idx[i]) for i in order]
    vals = [float(vals[i]) for i in order]
    best = idx[int(np.argmin(vals))]
    dump("C2_lscv_h.json", {
        "config": "C2", "workload": "LSCV_h d=1, n=65536, MW#6 bimodal mixture, datagen seed 2, 1024-point grid",
        "cite": "PAPER.md P:259-342 (Eq. 20-28), P:402-449 (Eq. 36-41); grid reading Z4, ties Z5",
        "n_grid": 1024, "h0": oracle.lscv_h0(n, 1), "indices": idx, "h": [float(grid[k]) for k in idx],
        "g": vals, "argmin_index_among_evaluated": best,
        "note": "every 32nd grid point plus all points within +-24 of the coarse argmin",
        "oracle_seconds": time.time() - t0, "threads": THREADS})


def c3():
    X = datagen.config_data("C3")
    t0 = time.time()
    trace = []
    r = oracle.lscv_H_select(X, max_iter=500, tol=1e-7, threads=THREADS, trace=trace)
    dump("C3_lscv_H.json", {
        "config": "C3", "workload": "LSCV_H d=2, n=32768, correlated 2-component mixture, datagen seed 3",
        "cite": "PAPER.md P:346-397 (Eq. 29-35), Nelder-Mead reading Z8",
        "H_start": oracle.vech(r["H_start"]).tolist(), "vechH": r["x"].tolist(), "f": r["f"],
        "iterations": r["iterations"], "stop": r["stop"],
        "final_simplex": [v.tolist() for v in r["simplex"]], "final_fvals": list(map(float, r["fvals"])),
        "evaluations": len(trace), "oracle_seconds": time.time() - t0, "threads": THREADS})


def c5():
    n = 1 << 18
    X = datagen.config_data("C5")
    cands = datagen.c5_candidates(n, 256)
    pick = list(range(0, 256, 32))
    t0 = time.time()
    g = [oracle.lscv_H_score(X, cands[k], threads=THREADS) for k in pick]
    dump("C5_lscv_H.json", {
        "config": "C5", "workload": "LSCV_H d=4, n=2^18, 3-component mixture, datagen seed 5; 256 candidates",
        "cite": "PAPER.md P:368-389 (Eq. 30-34)", "candidate_recipe": "datagen.c5_candidates(n, 256)",
        "indices": pick, "vechH": [cands[k].tolist() for k in pick], "g": g,
        "oracle_seconds": time.time() - t0, "threads": THREADS})


def c4b():
    """A second n = 2^20 PLUGIN data set (MW#4 kurtotic, seed 14): the Psi-hat margin at C4 size
    on another shape (the C4 Psi4 error rested on one seed and one mixture)."""
    x = datagen.sample_mixture("kurtotic", 1 << 20, 14)[0]
    t0 = time.time()
    tr = oracle.plugin(x, threads=THREADS)
    dump("C4b_plugin.json", {
        "config": "C4b", "workload": "PLUGIN, n=2^20, Marron-Wand #4 kurtotic mixture, datagen seed 14",
        "cite": "PAPER.md P:203-256 (Sec. 4.4.1 steps 1-8, Eq. 11-18), reading Z1 for Eq. 15/17",
        "trace": tr, "oracle_seconds": time.time() - t0, "threads": THREADS})


def t2048():
    """Raw Psi_r pair sums on ragged n that the library evaluates with 2048-row tiles
    (n >= 128 x 2048): n = 2^18 + 37 (r = 4, 6, 8) and n = 300001 (r = 6), skewed mixture seed 8."""
    xs = datagen.sample_mixture("skewed", 300001, 8)[0]
    out = []
    t0 = time.time()
    for n, r, g in [((1 << 18) + 37, 4, 0.12), ((1 << 18) + 37, 6, 0.2), ((1 << 18) + 37, 8, 0.3),
                    (300001, 6, 0.18)]:
        S = oracle.psi_pairsum(xs[:n], r, g, threads=THREADS)
        out.append({"n": n, "r": r, "g": g, "S": S})
        print(out[-1], flush=True)
    dump("T2048_psi.json", {
        "config": "T2048", "workload": "raw Psi_r sums sum_{i<j} He_r(u) exp(-u^2/2), u = (x_i - x_j)/g, "
        "first n samples of datagen.sample_mixture('skewed', 300001, 8)",
        "cite": "PAPER.md P:227-247 (Eq. 15, 17 pair sums); tiling P:539-566", "cases": out,
        "oracle_seconds": time.time() - t0, "threads": THREADS})


def esc():
    """Raw Psi sums for the automatic-precision decision tests: skewed seed 7, n = 131109 at
    (r, g) = (8, 0.2) (kappa ~ 4e4: the fp32-term pass is re-run in fp64) and (6, 0.2) (kappa ~ 8e3:
    it is not)."""
    xs = datagen.sample_mixture("skewed", 131109, 7)[0]
    out = []
    t0 = time.time()
    for r, g in [(8, 0.2), (6, 0.2)]:
        out.append({"n": 131109, "r": r, "g": g, "S": oracle.psi_pairsum(xs, r, g, threads=THREADS)})
    dump("ESC_psi.json", {
        "config": "ESC", "workload": "raw Psi_r sums, datagen.sample_mixture('skewed', 131109, 7)",
        "cite": "PAPER.md P:227-247 (Eq. 15, 17 pair sums)", "cases": out,
        "oracle_seconds": time.time() - t0, "threads": THREADS})


def c5small():
    """All 256 C5 candidates at n = 4096."""
    n = 4096
    X = datagen.config_data("C5", n=n)
    cands = datagen.c5_candidates(n, 256)
    t0 = time.time()
    g = [oracle.lscv_H_score(X, c, threads=THREADS) for c in cands]
    dump("C5small_lscv_H.json", {
        "config": "C5small", "workload": "LSCV_H d=4, n=4096 (datagen.config_data('C5', n=4096)), all 256 "
        "candidates datagen.c5_candidates(4096, 256)", "cite": "PAPER.md P:368-389 (Eq. 30-34)",
        "g": g, "oracle_seconds": time.time() - t0, "threads": THREADS})


def f1():
    """LSCV_h at d = 2 and 4 on the F1 workload (bench_configs F1: n = 65536, C5 mixture's first d
    coordinates), six h of its 1024-point grid (row f1)."""
    grid = np.linspace(0.05, 1.5, 1024)
    idx = [0, 31, 100, 300, 700, 1023]
    out = {}
    t0 = time.time()
    for d in (2, 4):
        X = datagen.config_data("C5", n=65536)[:d]
        out[str(d)] = {"h": [float(grid[k]) for k in idx], "indices": idx,
                       "g": [float(v) for v in oracle.lscv_h_scores(X, grid[idx], threads=THREADS)]}
    dump("F1_lscv_h.json", {
        "config": "F1", "workload": "LSCV_h d=2 and d=4, n=65536 (datagen.config_data('C5', n=65536)[:d]), "
        "grid np.linspace(0.05, 1.5, 1024)", "cite": "PAPER.md P:308-322 (Eq. 24), P:402-449 (Eq. 36-41)",
        "cases": out, "oracle_seconds": time.time() - t0, "threads": THREADS})


def f2():
    """KDE evaluation at full F2 size on sampled queries (row f2): n = 2^20 C4 samples, d = 1, h = 0.05,
    64 of the 2^16 linspace(-3, 4) queries; n = 32768 C3 samples, d = 2, 64 of the 2^15 C3 queries."""
    t0 = time.time()
    x = datagen.config_data("C4")
    y = np.linspace(-3, 4, 1 << 16)
    qi = list(range(0, 1 << 16, 1024))
    f1d = oracle.kde_eval(x, y[qi][None, :], [0.05 ** 2])
    X = datagen.config_data("C3")
    Y = datagen.sample_mixture("C3", 1 << 15, 99)
    qj = list(range(0, 1 << 15, 512))
    f2d = oracle.kde_eval(X, Y[:, qj], [0.012, 0.002, 0.011])
    dump("F2_eval.json", {
        "config": "F2", "workload": "fhat at sampled queries: d=1 C4 samples (n=2^20), H=[0.05^2], queries "
        "np.linspace(-3, 4, 2^16)[::1024]; d=2 C3 samples (n=32768), vechH=[0.012, 0.002, 0.011], queries "
        "datagen.sample_mixture('C3', 2^15, 99)[:, ::512]", "cite": "PAPER.md P:114-140 (Eq. kde-def-H, K_H)",
        "d1": {"query_index": qi, "f": [float(v) for v in f1d]}, "d2": {"query_index": qj, "f": [float(v) for v in f2d]},
        "oracle_seconds": time.time() - t0})


if __name__ == "__main__":
    which = sys.argv[1:] or ["C1", "C4", "C2", "C3", "C5"]
    for w in which:
        print("golden", w, flush=True)
        {"C1": c1, "C4": c4, "C2": c2, "C3": c3, "C5": c5, "C4b": c4b, "T2048": t2048,
         "C5small": c5small, "ESC": esc, "F1": f1, "F2": f2}[w]()
