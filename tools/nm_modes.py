"""Time the LSCV_H Nelder-Mead selector in speculative (4 candidates per round) and serial
(1-2 per round) mode on C3 (and a d = 4 sample): wall time, GPU launches, evaluations."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1505_01998_b200 as kb  # noqa: E402

ctx = kb.Context(profiling=True)
for name, X in (("C3", datagen.config_data("C3")), ("C5 d=4 n=32768", datagen.config_data("C5", n=32768))):
    Xd = kb.to_device(X)
    for spec in (1, 0):
        best = None
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = ctx.select_bandwidth(kb.LSCV_H, Xd, speculative=spec)
            dt = (time.perf_counter() - t0) * 1e3
            if best is None or dt < best[0]:
                best = (dt, r, ctx.last_profile())
        dt, r, p = best
        print(json.dumps({"data": name, "speculative": spec, "wall_ms": dt, "pair_ms": p["pair_ms"],
                          "launches": p["pair_launches"], "evaluations": r["evaluations"],
                          "iterations": r["iterations"], "objective": r["objective"],
                          "vechH": r["vechH"].tolist()}), flush=True)
