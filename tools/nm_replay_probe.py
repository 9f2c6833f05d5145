"""Device Nelder-Mead graph build / replay across changing problem shapes (memcheck probe).
python tools/nm_replay_probe.py [seq]   seq = comma list of mix:n:d:seed:max_iter"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, datagen, paper_1505_01998_b200 as kb  # noqa: E402
seq = sys.argv[1] if len(sys.argv) > 1 else "C3:3000:2:41:500,C3:700:2:42:40,C5:1200:3:43:500"
ctx = kb.Context()
for item in seq.split(","):
    mix, n, d, seed, it = item.split(":")
    X = datagen.sample_mixture(mix, int(n), int(seed))[: int(d)]
    Xd = kb.to_device(X)
    a = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=int(it), nm_loop=0)
    if os.environ.get("HOSTLOOP", "1") == "1":
        ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=int(it), nm_loop=1)
    c = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=int(it), nm_loop=0)
    print(item, a["objective"], c["objective"], flush=True)
