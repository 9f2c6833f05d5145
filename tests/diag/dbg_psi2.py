import math, sys, os
import numpy as np
sys.path.insert(0, os.getcwd())
import datagen, oracle
import paper_1505_01998_b200 as kb
ctx = kb.Context()
s2p = math.sqrt(2*math.pi)
n = int(sys.argv[1]); g = float(sys.argv[2])
x = datagen.sample_mixture("skewed", 64*2048+37, 7)[:, :n]
got = kb.fixed_value(ctx.raw_sums(kb.SUM_PSI6, kb.to_device(x), [g])[0]) / s2p
cache = f"scratch/ref_{n}_{g}.npy"
ref = float(np.load(cache)) if os.path.exists(cache) else oracle.psi_pairsum(x[0], 6, g, threads=16)
np.save(cache, ref)
print(os.environ.get("KDE_DEBUG_PSI_TILE"), n, g, got, ref, (got-ref)/abs(ref), flush=True)
