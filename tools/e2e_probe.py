"""Where does the end-to-end time of one C4 PLUGIN step go?  (GPU diagnostic, not a bench.)

Times, per step: CUDA-event device time of kde_plugin_h on resident data, host wall time of the
same call, and host wall time including the pinned H2D copy, with profiling on and off.
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_1505_01998_b200 as kb  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    x = datagen.config_data("C4", n=n)
    xd = kb.to_device(x)
    xp = torch.from_numpy(x).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    for prof in (True, False):
        ctx = kb.Context(device=0, profiling=prof)
        for _ in range(3):
            ctx.plugin_h(xd)
        rows = []
        for _ in range(5):
            flush.random_(0, 255)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(s)
            ctx.plugin_h(xd)
            e1.record(s)
            e1.synchronize()
            wall = (time.perf_counter() - t0) * 1e3
            flush.random_(0, 255)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            y = xp.to("cuda", non_blocking=True)
            t2 = time.perf_counter()
            ctx.plugin_h(y)
            t3 = time.perf_counter()
            rows.append({"dev_ms": e0.elapsed_time(e1), "wall_ms": wall, "e2e_ms": (t3 - t1) * 1e3,
                         "h2d_enqueue_ms": (t2 - t1) * 1e3,
                         "pair_ms": ctx.last_profile()["pair_ms"] if prof else None})
        print(json.dumps({"profiling": prof, "n": n, "steps": rows}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
