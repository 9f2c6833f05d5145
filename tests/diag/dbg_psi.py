import math, sys, time, os
import numpy as np
sys.path.insert(0, os.getcwd())
import datagen, oracle
import paper_1505_01998_b200 as kb
ctx = kb.Context()
s2p = math.sqrt(2*math.pi)
n = 64*2048+37; g = 0.2
x = datagen.sample_mixture("skewed", n, 7)
ref = float(np.fromfile('scratch/ref131k.bin')[0]) if os.path.exists('scratch/ref131k.bin') else oracle.psi_pairsum(x[0], 6, g, threads=16)
print("ref", ref, flush=True)
for n2 in [n, 20000, 5000]:
    xx = x[:, :n2]
    r2 = ref if n2 == n else oracle.psi_pairsum(xx[0], 6, g, threads=16)
    for T in ["512", "2048"]:
        os.environ["KDE_DEBUG_PSI_TILE"] = T
        # tile_for caches the env at first call: use a fresh process per T instead
    print(n2, "ref", r2, flush=True)
