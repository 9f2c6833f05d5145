"""memcheck probe: a context with a caller workspace, then another context's device Nelder-Mead
build + replay (tools/nm_memcheck_probe.py none|plain|ws; env KEEP_C1, NO_HOST)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, datagen, paper_1505_01998_b200 as kb
mode = sys.argv[1]
X = datagen.sample_mixture("C3", 4000, 23)
c1 = kb.Context()
if mode == "ws":
    ws = torch.full((kb.lib().kde_workspace_bytes(4000, 2, 64),), 255, dtype=torch.uint8, device="cuda")
    c1.set_workspace(ws)
if mode != "none":
    c1.select_bandwidth(kb.LSCV_H, X, max_iter=60, nm_starts=4)
if not os.environ.get("KEEP_C1"):
    c1.close()
ctx = kb.Context()
X2 = datagen.sample_mixture("C3", 3000, 41)[:2]; Xd = kb.to_device(X2)
a = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=500, nm_loop=0)
if not os.environ.get("NO_HOST"):
    b = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=500, nm_loop=1)
c = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=500, nm_loop=0)
print(mode, a["objective"], c["objective"])
