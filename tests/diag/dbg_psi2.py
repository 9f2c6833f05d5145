"""Psi_6 raw sum at (n, g) vs the fp64 oracle: python tests/diag/dbg_psi2.py N G (GPU diagnostic)."""
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
cache = f"/tmp/kde_psiref_{n}_{g}.npy"   # per-machine cache of the oracle value
ref = float(np.load(cache)) if os.path.exists(cache) else oracle.psi_pairsum(x[0], 6, g, threads=16)
np.save(cache, ref)
print(os.environ.get("KDE_DEBUG_PSI_TILE"), n, g, got, ref, (got-ref)/abs(ref), flush=True)
