"""Time every BASELINE.json config through the public API (1 GPU), one JSON line each
(SURVEY §8(d) d8 report).

  python tools/bench_configs.py [C1 C2 C3 C4 C5 ...] [--reps 3]

evals = algorithmic pair-kernel evaluations (pairs i<j x candidates); pair_ms = device time of
the pair-kernel launches (library events); wall_ms = host wall time of the call (time to
bandwidth / to scores, X resident on the device).  MUFU peak = 16 EX2/clk/SM x SMs x 1965 MHz.
`parity` compares with the fp64 oracle's stored values in tests/golden/*.json (written by
tests/golden/make_golden.py, which calls only oracle/; this tool never runs the oracle).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1505_01998_b200 as kb  # noqa: E402

SMS = torch.cuda.get_device_properties(0).multi_processor_count
PEAK = 16 * SMS * 1965e6


_CLOCKS = {}


def timed(fn, reps, warm=True):
    """Best of `reps` calls (after one untimed warm-up call when warm); the SM clock is sampled by
    nvidia-smi during the timed calls (bench.ClockSampler) and reported by line()."""
    from bench import ClockSampler
    if warm:
        fn()
    best = None
    cs = ClockSampler(0)
    cs.start()
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        prof = ctx.last_profile()
        if best is None or dt < best[0]:
            best = (dt, prof, out)
    _CLOCKS.clear()
    _CLOCKS.update(cs.stop())
    return best


GOLD = os.path.join(ROOT, "tests", "golden")


def gold(name):
    return json.load(open(os.path.join(GOLD, name)))


def relerr(a, b):
    return abs(a - b) / abs(b)


def sm_clock():
    try:
        import subprocess
        out = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=10).stdout.strip()
        return float(out.split()[0])
    except Exception:
        return None


def line(cfg, what, dt, prof, extra=None, alg=None):
    # evals = evaluated pair-kernel evaluations (the library's profile leaves out the pairs of tiles
    # skipped as exactly zero); alg = algorithmic evaluations (all pairs x candidates), when known
    ev = prof["pair_evals"]
    clk = dict(_CLOCKS) if _CLOCKS.get("sm_mhz") else {"sm_mhz": sm_clock(), "reasons": ["sampled after the call"]}
    d = {"config": cfg, "what": what, "gpus": 1, "sm_clock_mhz": clk.get("sm_mhz"), "clocks": clk,
         "wall_ms": dt * 1e3, "pair_ms": prof["pair_ms"],
         "pair_launches": prof["pair_launches"], "evals": ev,
         "evals_per_s_pair": ev / (prof["pair_ms"] / 1e3) if prof["pair_ms"] > 0 else None,
         "frac_mufu_peak": (ev / (prof["pair_ms"] / 1e3)) / PEAK if prof["pair_ms"] > 0 else None}
    if alg is not None:
        d.update({"evals_algorithmic": alg, "evaluated_fraction": ev / alg,
                  "algorithmic_evals_per_s_wall": alg / dt})
    if extra:
        d.update(extra)
    print(json.dumps(d), flush=True)


ctx = kb.Context(profiling=True)


def run(cfg, reps):
    if cfg == "C1":
        x = kb.to_device(datagen.config_data("C1"))
        dt, prof, out = timed(lambda: ctx.plugin_h(x), reps)
        g = gold("C1_plugin.json")["trace"]
        line(cfg, "plugin_h n=1000", dt, prof, {"n": 1000, "d": 1, "n_cand": 2, "h": out[0],
             "parity": {"reference": "tests/golden/C1_plugin.json (fp64 oracle)",
                        "rel_err": {k: relerr(out[1][k], g[k]) for k in ("psi6", "psi4", "h")}}})
    elif cfg == "C4":
        x = kb.to_device(datagen.config_data("C4"))
        dt, prof, out = timed(lambda: ctx.plugin_h(x), reps)
        g = gold("C4_plugin.json")["trace"]
        line(cfg, "plugin_h n=2^20", dt, prof, alg=2 * (1 << 20) * ((1 << 20) - 1) / 2, extra={"n": 1 << 20, "d": 1, "n_cand": 2, "h": out[0], "trace": out[1],
             "parity": {"reference": "tests/golden/C4_plugin.json (fp64 oracle)",
                        "rel_err": {k: relerr(out[1][k], g[k]) for k in ("psi6", "psi4", "h")}}})
    elif cfg == "C2":
        X = datagen.config_data("C2")
        Xd = kb.to_device(X)
        n = X.shape[1]
        h0 = (4.0 / (3.0 * n)) ** 0.2
        grid = np.linspace(h0 / 4, 4 * h0, 1024)
        dt, prof, g = timed(lambda: ctx.lscv_h_scores(Xd, grid), reps)
        pairs = n * (n - 1) / 2
        # a quarter of the exponentials come from the FMA pipe, so the kernel's own bound is
        # the MUFU peak / 0.75 (21.3 evals/clk/SM)
        mixed = PEAK / 0.75
        eps = prof["pair_evals"] / (prof["pair_ms"] / 1e3) if prof["pair_ms"] > 0 else 0.0
        line(cfg, "lscv_h_scores 1024 h, n=65536", dt, prof, {"argmin": int(np.argmin(g)), "g_min": float(g.min()),
             "mixed_bound_evals_per_s": mixed, "frac_mixed_bound": eps / mixed}, alg=pairs * 1024)
        dt, prof, r = timed(lambda: ctx.select_bandwidth(kb.LSCV_h, Xd, n_grid=1024), 1)
        gd = gold("C2_lscv_h.json")
        gs = ctx.lscv_h_scores(Xd, gd["h"])
        line(cfg, "select LSCV_h (1024-point grid)", dt, prof, {"n": n, "d": 1, "n_cand": 1024, "h": r["h"],
             "index": r["iterations"],
             "parity": {"reference": "tests/golden/C2_lscv_h.json (fp64 oracle, 81 grid points)",
                        "max_rel_err": float(np.max(np.abs(gs - np.array(gd["g"])) / np.abs(gd["g"]))),
                        "argmin_match": r["iterations"] == gd["argmin_index_among_evaluated"]}}, alg=pairs * 1024)
    elif cfg == "C3":
        X = datagen.config_data("C3")
        Xd = kb.to_device(X)
        gd = gold("C3_lscv_H.json")
        host_pair_ms = None
        for loop in (1, 0):   # host loop first: its pair_ms is the pair-kernel time alone
            dt, prof, r = timed(lambda: ctx.select_bandwidth(kb.LSCV_H, Xd, nm_loop=loop), reps)
            if loop == 1:
                host_pair_ms = prof["pair_ms"]
            Hg, Ho = datagen.unvech(r["vechH"], 2), datagen.unvech(np.array(gd["vechH"]), 2)
            extra = {"n": X.shape[1], "d": 2, "vechH": r["vechH"].tolist(), "objective": r["objective"],
                     "iterations": r["iterations"], "evaluations": r["evaluations"], "stop": r["stop_reason"],
                     "nm_loop": "device (one CUDA graph, conditional WHILE)" if loop == 0 else "host (sync per round)",
                     "pair_kernel_ms_host_loop": host_pair_ms,
                     "wall_over_pair_kernel_time": dt * 1e3 / host_pair_ms if host_pair_ms else None,
                     "parity": {"reference": "tests/golden/C3_lscv_H.json (fp64 oracle Nelder-Mead)",
                                "same_iterations": r["iterations"] == gd["iterations"],
                                "H_rel_diff": float(np.max(np.abs(Hg - Ho)) / np.max(np.diag(Ho))),
                                "objective_rel_diff": relerr(r["objective"], gd["f"])}}
            line(cfg, f"select LSCV_H (Nelder-Mead, {'device' if loop == 0 else 'host'} loop)", dt, prof, extra,
                 alg=r["evaluations"] * X.shape[1] * (X.shape[1] - 1) / 2)
    elif cfg == "F3":
        # the paper's two-phase LSCV_h on the C2 workload: HBM-bound phase 2 at 1 h per pass
        X = datagen.config_data("C2")
        Xd = kb.to_device(X)
        n = X.shape[1]
        h0 = (4.0 / (3.0 * n)) ** 0.2
        grid = np.linspace(h0 / 4, 4 * h0, 1024)
        T = 256
        tiles = ((n + T - 1) // T) * ((n + T - 1) // T + 1) // 2
        buf_bytes = tiles * T * T * 4
        for B in (1, 4, 16):
            dt, prof, g = timed(lambda: ctx.lscv_h_scores_materialized(Xd, grid, h_per_pass=B), 2)
            passes = (1024 + B - 1) // B
            gbs = buf_bytes * passes / (prof["pair_ms"] / 1e3) / 1e9
            line(cfg, f"materialised S(v) LSCV_h, 1024 h, {B} h per pass", dt, prof,
                 {"phase1_ms": ctx.last_aux_ms(), "buffer_GB": buf_bytes / 1e9, "phase2_hbm_GBps": gbs,
                  "hbm_frac_of_measured_copy": gbs / 6552.0, "hbm_frac_of_nominal_7700": gbs / 7700.0, "argmin": int(np.argmin(g))})
    elif cfg == "F1":
        # LSCV_h for d > 1 (whitened scalar h, row f1): n = 65536, 1024 h, d = 2 and 4
        for d in (2, 4):
            X = datagen.config_data("C5", n=65536)[:d]
            Xd = kb.to_device(X)
            grid = np.linspace(0.05, 1.5, 1024)
            dt, prof, g = timed(lambda: ctx.lscv_h_scores(Xd, grid), reps)
            line(cfg, f"lscv_h_scores d={d}, n=65536, 1024 h", dt, prof, {"argmin": int(np.argmin(g))})
    elif cfg == "F4":
        # optimizer variants: LSCV_h 150-point grid + 6 refinement sections vs the 1024 grid (C2),
        # and 4-start lockstep Nelder-Mead for LSCV_H (C3)
        X = datagen.config_data("C2")
        Xd = kb.to_device(X)
        dt, prof, r = timed(lambda: ctx.select_bandwidth(kb.LSCV_h, Xd, n_grid=150, refine_steps=6), 1)
        line(cfg, "select LSCV_h, 150-point grid + 6 x 16-point refinement (C2 data)", dt, prof,
             {"h": r["h"], "objective": r["objective"], "evaluations": r["evaluations"], "steps": r["stop_reason"]})
        X = datagen.config_data("C3")
        Xd = kb.to_device(X)
        for K in (1, 4):
            dt, prof, r = timed(lambda: ctx.select_bandwidth(kb.LSCV_H, Xd, nm_starts=K), reps)
            line(cfg, f"select LSCV_H, {K}-start Nelder-Mead (C3)", dt, prof,
                 {"vechH": r["vechH"].tolist(), "objective": r["objective"], "iterations": r["iterations"],
                  "evaluations": r["evaluations"]})
    elif cfg == "F2":
        # KDE evaluation: n = 2^20 samples (C4 data) at m = 2^16 queries, d = 1; and d = 2 (C3)
        x = datagen.config_data("C4")
        y = np.linspace(-3, 4, 1 << 16)[None, :]
        xd, yd = kb.to_device(x), kb.to_device(y)
        dt, prof, f = timed(lambda: ctx.evaluate(xd, yd, [0.05 ** 2]), reps)
        line(cfg, "evaluate fhat, d=1, n=2^20 samples, m=2^16 queries", dt, prof)
        X = datagen.config_data("C3")
        Y = datagen.sample_mixture("C3", 1 << 15, 99)
        Xd, Yd = kb.to_device(X), kb.to_device(Y)
        dt, prof, f = timed(lambda: ctx.evaluate(Xd, Yd, [0.012, 0.002, 0.011]), reps)
        line(cfg, "evaluate fhat, d=2, n=32768 samples, m=32768 queries", dt, prof)
        lo = np.linspace(-3, 3, 64)
        dt, prof, out = timed(lambda: ctx.aqp_1d(xd, 0.05, lo, lo + 0.5), reps)
        print(json.dumps({"config": cfg, "what": "aqp_1d 64 ranges, n=2^20", "wall_ms": dt * 1e3}), flush=True)
    elif cfg in ("C5", "C5P"):
        # C5P: the first 16 of the 256 candidates (same kernel, short enough for ncu --set full)
        n = 1 << 18
        X = datagen.config_data("C5")
        Xd = kb.to_device(X)
        cands = datagen.c5_candidates(n, 256)[: 16 if cfg == "C5P" else 256]
        dt, prof, g = timed(lambda: ctx.lscv_H_scores(Xd, cands), reps)
        # d = 4 is FMA-bound: per eval, on data whitened by the candidate, 4 sub +
        # 4 (sum of squares) + 2 (accumulate) FP32 lane-ops at the measured 125 FP32 lane-ops/clk/SM
        # (tools/pipes.cu)
        fma_peak = 125.0 / (2 * 4 + 2) * SMS * 1965e6
        ev = prof["pair_evals"] / (prof["pair_ms"] / 1e3)
        extra = {"n": n, "d": 4, "n_cand": len(cands), "g_first": g[:4].tolist(),
                 "fma_bound_evals_per_s": fma_peak, "frac_fma_bound": ev / fma_peak}
        if cfg == "C5":
            gd = gold("C5_lscv_H.json")
            extra["parity"] = {"reference": "tests/golden/C5_lscv_H.json (fp64 oracle, 8 of 256 candidates)",
                               "max_rel_err": float(np.max(np.abs(g[gd["indices"]] - np.array(gd["g"])) / np.abs(gd["g"])))}
        line(cfg, f"lscv_H_scores {len(cands)} H, d=4, n=2^18", dt, prof, extra, alg=len(cands) * n * (n - 1) / 2)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    reps = 3
    if "--reps" in sys.argv:
        reps = int(sys.argv[sys.argv.index("--reps") + 1])
    for cfg in args or ["C1", "C4", "C2", "C5", "C3"]:
        run(cfg, reps)
