"""C3 (LSCV_H d=2, n=32768) Nelder-Mead select through the public API, device loop (default) or host
loop (--host): prints wall time; used under ncu for the per-kernel durations of one search."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, datagen, paper_1505_01998_b200 as kb
ctx = kb.Context()
Xd = kb.to_device(datagen.config_data("C3"))
loop = 1 if "--host" in sys.argv else 0
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 1
for _ in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = ctx.select_bandwidth(kb.LSCV_H, Xd, nm_loop=loop)
    torch.cuda.synchronize(); print("wall_ms %.3f iterations %d evals %d" % ((time.perf_counter() - t0) * 1e3, r["iterations"], r["evaluations"]))
