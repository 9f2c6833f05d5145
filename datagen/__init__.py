"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no kernels, no sums, no bandwidth formulas);
it only draws samples.  Both sides of every parity test read the same bytes from here.

Generator: a counter-based splitmix64 stream.  Draw k of stream `seed`
is splitmix64_mix(seed * 2**32 + 0x9E3779B97F4A7C15 * (k + 1)) — every draw is a pure
function of (seed, k), so arrays are reproducible in any order / chunking.  A uniform is
u = ((z >> 11) + 0.5) * 2**-53 in (0, 1), a standard normal is Box–Muller on two uniforms
(cos branch only).  Mixture component for a sample: first l with u_c < cumulative weight.

Workloads (the paper's experiments used unspecified "random" data; shapes
follow BASELINE.json configs):
  C1  N(0,1), n=1000, d=1                                              seed 1
  C2  Marron–Wand #6 bimodal ½N(−1,(2/3)²)+½N(1,(2/3)²), n=65536       seed 2
  C3  d=2 correlated mixture (see MIXTURES['C3']), n=32768             seed 3
  C4  Marron–Wand #2 skewed ⅕N(0,1)+⅕N(½,(⅔)²)+⅗N(13/12,(5/9)²), n=2^20 seed 4
  C5  d=4 3-component mixture, covariances AAᵀ/4+0.1I (A~N(0,1), stream 5), n=2^18 seed 5
Layout: X is d×n, row-major (each dimension a contiguous row, Eq. 19).
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, k0: int, count: int) -> np.ndarray:
    """Draws k0 .. k0+count-1 of stream `seed` as uint64."""
    with np.errstate(over="ignore"):
        k = np.arange(k0 + 1, k0 + 1 + count, dtype=np.uint64)
        z = np.uint64((seed << 32) & 0xFFFFFFFFFFFFFFFF) + k * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniforms(seed: int, k0: int, count: int) -> np.ndarray:
    z = splitmix64(seed, k0, count)
    return ((z >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def normals(seed: int, k0: int, count: int) -> np.ndarray:
    """Standard normals from draws 2*k0 .. of the stream (Box–Muller, cos branch)."""
    u = uniforms(seed, 2 * k0, 2 * count)
    u1, u2 = u[0::2], u[1::2]
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


# Mixture recipes: (weights, means[l][d], covariances[l][d][d]).  C5 covariances are drawn.
def _c5_recipe():
    d = 4
    w = [0.5, 0.3, 0.2]
    e = np.eye(d)
    means = [1.5 * e[0], 1.5 * e[1], 1.5 * (-e[0] - e[1])]
    covs = []
    for l in range(3):
        a = normals(5, 1_000_000_000 + 16 * l, d * d).reshape(d, d)
        covs.append(a @ a.T / 4.0 + 0.1 * np.eye(d))
    return w, [np.asarray(m, float) for m in means], covs


MIXTURES = {
    "N01": ([1.0], [np.zeros(1)], [np.eye(1)]),
    "bimodal": ([0.5, 0.5], [np.array([-1.0]), np.array([1.0])],
                [np.array([[4.0 / 9.0]]), np.array([[4.0 / 9.0]])]),
    "skewed": ([0.2, 0.2, 0.6], [np.array([0.0]), np.array([0.5]), np.array([13.0 / 12.0])],
               [np.array([[1.0]]), np.array([[4.0 / 9.0]]), np.array([[25.0 / 81.0]])]),
    # Marron–Wand #4 kurtotic unimodal: ⅔N(0,1) + ⅓N(0,(1/10)²) (second n=2^20 PLUGIN golden)
    "kurtotic": ([2.0 / 3.0, 1.0 / 3.0], [np.array([0.0]), np.array([0.0])],
                 [np.array([[1.0]]), np.array([[0.01]])]),
    "C3": ([0.5, 0.5], [np.array([-1.0, -1.0]), np.array([1.0, 1.0])],
           [4.0 / 9.0 * np.array([[1.0, 0.7], [0.7, 1.0]]),
            4.0 / 9.0 * np.array([[1.0, -0.5], [-0.5, 1.0]])]),
}


def mixture(name: str):
    if name == "C5":
        return _c5_recipe()
    return MIXTURES[name]


def sample_mixture(name: str, n: int, seed: int) -> np.ndarray:
    """n samples of mixture `name` as a d×n fp64 row-major array."""
    w, means, covs = mixture(name)
    d = len(means[0])
    uc = uniforms(seed, 0, n)                      # component selector draws
    z = normals(seed, n, n * d).reshape(n, d)      # disjoint draws of the same stream
    cw = np.cumsum(w)
    cw[-1] = 1.0 + 1e-12
    comp = np.searchsorted(cw, uc, side="right")
    X = np.empty((d, n), dtype=np.float64)
    for l in range(len(w)):
        idx = np.nonzero(comp == l)[0]
        if idx.size == 0:
            continue
        c = np.linalg.cholesky(np.asarray(covs[l], float))   # sampling transform only
        X[:, idx] = (np.asarray(means[l], float)[:, None] + c @ z[idx].T)
    return np.ascontiguousarray(X)


CONFIGS = {
    # name: (mixture, n, seed, d)
    "C1": ("N01", 1000, 1, 1),
    "C2": ("bimodal", 65536, 2, 1),
    "C3": ("C3", 32768, 3, 2),
    "C4": ("skewed", 1 << 20, 4, 1),
    "C5": ("C5", 1 << 18, 5, 4),
}


def config_data(name: str, n: int | None = None, seed: int | None = None) -> np.ndarray:
    mix, n0, s0, _ = CONFIGS[name]
    return sample_mixture(mix, n0 if n is None else n, s0 if seed is None else seed)


def population_covariance(name: str) -> np.ndarray:
    """Covariance of the mixture distribution from its recipe constants (no sample data)."""
    w, means, covs = mixture(name)
    mu = sum(wi * m for wi, m in zip(w, means))
    S = sum(wi * (np.asarray(c) + np.outer(m, m)) for wi, m, c in zip(w, means, covs))
    return S - np.outer(mu, mu)


def c5_candidates(n: int, count: int = 256, name: str = "C5") -> np.ndarray:
    """Candidate SPD bandwidth matrices for the C5 batch, as vech rows.

    H_k = s_k R_kᵀ H_ref R_k with H_ref = (4/(d+2))^{2/(d+4)} n^{-2/(d+4)} Σ_pop (normal-scale
    reference built from the recipe's population covariance, not from the sample), s_k geometric
    in [0.5, 2], R_k a product of seeded Givens rotations with angles ≤ 0.3 rad.
    """
    S = population_covariance(name)
    d = S.shape[0]
    Href = (4.0 / (d + 2)) ** (2.0 / (d + 4)) * n ** (-2.0 / (d + 4)) * S
    out = np.empty((count, d * (d + 1) // 2))
    ang = (uniforms(77, 0, count * d * d) * 2.0 - 1.0) * 0.3
    for k in range(count):
        s = 0.5 * 4.0 ** (k / max(count - 1, 1))
        R = np.eye(d)
        t = 0
        for a in range(d):
            for b in range(a + 1, d):
                G = np.eye(d)
                c_, s_ = np.cos(ang[k * d * d + t]), np.sin(ang[k * d * d + t])
                G[a, a] = c_; G[b, b] = c_; G[a, b] = -s_; G[b, a] = s_
                R = R @ G
                t += 1
        H = s * R.T @ Href @ R
        H = 0.5 * (H + H.T)
        out[k] = vech(H)
    return out


def vech(A: np.ndarray) -> np.ndarray:
    """Stack the lower triangle column by column (Eq. vech)."""
    d = A.shape[0]
    return np.array([A[i, j] for j in range(d) for i in range(j, d)])


def unvech(v, d: int) -> np.ndarray:
    A = np.empty((d, d))
    t = 0
    for j in range(d):
        for i in range(j, d):
            A[i, j] = A[j, i] = v[t]
            t += 1
    return A
