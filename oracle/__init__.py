"""TEST INFRASTRUCTURE ONLY — the fp64 CPU oracle for arxiv 1505.01998's bandwidth selectors.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this package.  It shares no code with the CUDA path (paper_1505_01998_b200/) and never
imports it.  The O(n^2) sums live in kde_oracle.c (plain double loops, libm exp, Neumaier
sums); the O(1)/O(d^3) scalar chains, the small linear algebra and Nelder–Mead are written
here in plain Python floats (IEEE fp64), each following the cited passage of PAPER.md
(P:NNN = /root/reference/PAPER.md line NNN).

Parity status: every function below is pinned by tests/test_oracle_*.py against something
other than itself (quadrature identities, library routines, closed forms, invariants, MC
expectations); nelder_mead is pinned step for step to scipy's Nelder–Mead.  The PLUGIN chain
(every step of Eq. 11-18) is pinned to the mpmath X=[1,2,3] trace, lscv_h0 at d = 1, 2, 3 to
Eq. 25 simplified by hand, initial_simplex to hand-written vertices (reading Z8) and the
nm_starts 4^-k scaling to the evaluation trace (tests/test_paper_examples.py).  The GPU selector's
NM decision path is checked against this one by replay (tests/test_gpu_nm_replay.py: identical
decisions on seeded inputs); where an fp32-term objective could legitimately flip a near-tie
comparison, the SURVEY §8(c) c5 tie rule applies.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kde_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

PENALTY = 1e300


def build(force: bool = False) -> str:
    """Compile the C part with gcc (plain -O2, no fast-math: IEEE semantics kept)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC",
                               "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int64)
        i64, i32, f64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.oracle_hermite.argtypes = [i32, f64]; L.oracle_hermite.restype = f64
        L.oracle_kernel_deriv.argtypes = [i32, f64]; L.oracle_kernel_deriv.restype = f64
        L.oracle_psi_pairsum_rows.argtypes = [dp, i64, i32, f64, i64, i64, dp]
        L.oracle_psi_r.argtypes = [dp, i64, i32, f64, dp]
        L.oracle_lscv_h_pairsums_rows.argtypes = [dp, i64, i32, dp, f64, i64, i64, dp]
        L.oracle_lscv_H_pairsums_rows.argtypes = [dp, i64, i32, dp, i64, i64, dp]
        L.oracle_lscv_h_modified.argtypes = [dp, i64, i32, dp, f64, dp, i32, dp]
        L.oracle_mean_cov.argtypes = [dp, i64, i32, dp, dp]
        L.oracle_tile_enumerate.argtypes = [i64, ip, ip]
        L.oracle_kde_eval.argtypes = [dp, i64, i32, dp, i64, dp, f64, dp]
        for f in ("oracle_psi_pairsum_rows", "oracle_psi_r", "oracle_lscv_h_pairsums_rows",
                  "oracle_lscv_H_pairsums_rows", "oracle_lscv_h_modified", "oracle_mean_cov",
                  "oracle_tile_enumerate", "oracle_kde_eval"):
            getattr(L, f).restype = i32
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _as_X(X) -> np.ndarray:
    X = np.ascontiguousarray(np.asarray(X, dtype=np.float64))
    if X.ndim == 1:
        X = X[None, :]
    return X


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle: {what} failed (rc={rc})")


# --------------------------------------------------------------------------- row splitting
def row_chunks(n: int, parts: int):
    """Split rows 0..n-1 into `parts` contiguous ranges of ~equal pair count (row i has n-1-i)."""
    total = n * (n - 1) // 2
    bounds, acc, target, i = [0], 0, 1, 0
    for i in range(n):
        acc += n - 1 - i
        while target < parts and acc >= total * target / parts:
            bounds.append(i + 1)
            target += 1
    while len(bounds) < parts + 1:
        bounds.append(n)
    bounds[-1] = n
    return [(bounds[k], bounds[k + 1]) for k in range(parts)]


def _parallel_rows(fn, n: int, threads: int, width: int):
    """Run fn(i0, i1) -> np.ndarray(width) over row chunks and add the parts in chunk order."""
    if threads <= 1:
        return fn(0, n)
    chunks = row_chunks(n, threads * 4)
    with ThreadPoolExecutor(max_workers=threads) as ex:
        parts = list(ex.map(lambda c: fn(*c), chunks))
    out = np.zeros(width)
    for p in parts:                      # fixed order
        out = out + p
    return out


# --------------------------------------------------------------------------- kernels
SQRT2PI = math.sqrt(2.0 * math.pi)


def hermite(r: int, u: float) -> float:
    return lib().oracle_hermite(r, u)


def kernel_deriv(r: int, u: float) -> float:
    """K^(r)(u) = He_r(u) exp(-u^2/2)/sqrt(2 pi)."""
    return lib().oracle_kernel_deriv(r, u)


def psi_pairsum(x, r: int, g: float, rows=None, threads: int = 1) -> float:
    """sum_{i<j} K^(r)((x_i - x_j)/g) over all pairs (or rows [i0,i1) with all j > i)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel())
    n = x.size
    L = lib()

    def fn(i0, i1):
        o = ctypes.c_double()
        _check(L.oracle_psi_pairsum_rows(_dp(x), n, r, g, i0, i1, ctypes.byref(o)), "psi sum")
        return np.array([o.value])

    if rows is not None:
        return float(fn(*rows)[0])
    return float(_parallel_rows(fn, n, threads, 1)[0])


def psi_r(x, r: int, g: float, threads: int = 1) -> float:
    """Psi_r-hat(g) = [2 S + n K^(r)(0)] / (n^2 g^(r+1))  (reading Z1)."""
    x = np.asarray(x, dtype=np.float64).ravel()
    n = x.size
    S = psi_pairsum(x, r, g, threads=threads)
    return (2.0 * S + n * kernel_deriv(r, 0.0)) / (n * n * g ** (r + 1))


def mean_cov(X):
    X = _as_X(X)
    d, n = X.shape
    m = np.zeros(d)
    C = np.zeros(d * d)
    _check(lib().oracle_mean_cov(_dp(X), n, d, _dp(m), _dp(C)), "mean_cov")
    return m, C.reshape(d, d)


# --------------------------------------------------------------------------- PLUGIN (Sec 4.4.1)
class DegenerateData(ValueError):
    pass


def plugin(x, threads: int = 1) -> dict:
    """Wand–Jones two-stage direct plug-in, steps 1-8 of P:203-256, in the paper's order."""
    x = np.asarray(x, dtype=np.float64).ravel()
    n = x.size
    if n < 2:
        raise ValueError("PLUGIN needs n >= 2")
    _, C = mean_cov(x[None, :])
    V = float(C[0, 0])                                   # step 1, Eq. 11 (two-pass, Z10)
    if not V > 0.0:
        raise DegenerateData("variance <= 0")
    sigma = math.sqrt(V)                                 # step 2, Eq. 12
    psi8ns = 105.0 / (32.0 * math.sqrt(math.pi) * sigma ** 9)   # step 3, Eq. 13
    K6_0 = -15.0 / SQRT2PI
    mu2 = 1.0
    g1 = (-2.0 * K6_0 / (mu2 * psi8ns * n)) ** (1.0 / 9.0)      # step 4, Eq. 14
    psi6 = psi_r(x, 6, g1, threads)                      # step 5, Eq. 15
    K4_0 = 3.0 / SQRT2PI
    if not psi6 < 0.0:
        raise ArithmeticError("Psi6 >= 0")
    g2 = (-2.0 * K4_0 / (mu2 * psi6 * n)) ** (1.0 / 7.0)        # step 6, Eq. 16
    psi4 = psi_r(x, 4, g2, threads)                      # step 7, Eq. 17
    if not psi4 > 0.0:
        raise ArithmeticError("Psi4 <= 0")
    RK = 1.0 / (2.0 * math.sqrt(math.pi))
    h = (RK / (mu2 ** 2 * psi4 * n)) ** 0.2              # step 8, Eq. 18
    return dict(V_hat=V, sigma_hat=sigma, psi8_ns=psi8ns, g1=g1, psi6=psi6, g2=g2,
                psi4=psi4, h=h)


# --------------------------------------------------------------------------- small linear algebra
def gauss_jordan(A):
    """Inverse and determinant by Gauss–Jordan elimination with partial pivoting."""
    A = [list(map(float, row)) for row in np.asarray(A, float)]
    d = len(A)
    I = [[1.0 if i == j else 0.0 for j in range(d)] for i in range(d)]
    det = 1.0
    for c in range(d):
        p = max(range(c, d), key=lambda r: abs(A[r][c]))
        if A[p][c] == 0.0:
            return None, 0.0
        if p != c:
            A[p], A[c] = A[c], A[p]
            I[p], I[c] = I[c], I[p]
            det = -det
        piv = A[c][c]
        det *= piv
        A[c] = [v / piv for v in A[c]]
        I[c] = [v / piv for v in I[c]]
        for r in range(d):
            if r != c and A[r][c] != 0.0:
                f = A[r][c]
                A[r] = [a - f * b for a, b in zip(A[r], A[c])]
                I[r] = [a - f * b for a, b in zip(I[r], I[c])]
    return np.array(I), det


def cholesky_pd(A, rel_tol: float = 1e-12):
    """Cholesky A = L L^T; returns None unless every pivot > rel_tol * max diag (PD test)."""
    A = np.asarray(A, float)
    d = A.shape[0]
    if not np.all(np.isfinite(A)) or np.any(A != A.T):
        return None
    mx = max(abs(A[i, i]) for i in range(d))
    L = [[0.0] * d for _ in range(d)]
    for j in range(d):
        s = A[j, j] - sum(L[j][k] ** 2 for k in range(j))
        if not s > rel_tol * mx:
            return None
        L[j][j] = math.sqrt(s)
        for i in range(j + 1, d):
            L[i][j] = (A[i, j] - sum(L[i][k] * L[j][k] for k in range(j))) / L[j][j]
    return np.array(L)


def jacobi_eigh(A, sweeps: int = 100):
    """Cyclic Jacobi eigendecomposition of a symmetric matrix: A = V diag(w) V^T."""
    A = np.array(A, dtype=float)
    d = A.shape[0]
    V = np.eye(d)
    for _ in range(sweeps):
        off = sum(A[i, j] ** 2 for i in range(d) for j in range(d) if i != j)
        if off == 0.0 or off < 1e-30 * sum(A[i, i] ** 2 for i in range(d)):
            break
        for p in range(d):
            for q in range(p + 1, d):
                if A[p, q] == 0.0:
                    continue
                theta = (A[q, q] - A[p, p]) / (2.0 * A[p, q])
                t = math.copysign(1.0, theta) / (abs(theta) + math.sqrt(theta * theta + 1.0))
                c = 1.0 / math.sqrt(t * t + 1.0)
                s = t * c
                J = np.eye(d)
                J[p, p] = c; J[q, q] = c; J[p, q] = s; J[q, p] = -s
                A = J.T @ A @ J
                V = V @ J
    return np.array([A[i, i] for i in range(d)]), V


def sqrtm_spd(S):
    """Symmetric square root via the eigendecomposition (reading Z9; the paper used ALGLIB)."""
    w, V = jacobi_eigh(S)
    if np.any(w <= 0):
        raise ValueError("matrix not positive definite")
    R = V @ np.diag(np.sqrt(w)) @ V.T
    return 0.5 * (R + R.T)


def vech(A):
    """Lower triangle stacked column by column."""
    A = np.asarray(A)
    d = A.shape[0]
    return np.array([A[i, j] for j in range(d) for i in range(j, d)])


def unvech(v, d: int):
    A = np.zeros((d, d))
    t = 0
    for j in range(d):
        for i in range(j, d):
            A[i, j] = A[j, i] = v[t]
            t += 1
    return A


def dim_from_vech(m: int) -> int:
    d = int(round((math.sqrt(8 * m + 1) - 1) / 2))
    if d * (d + 1) // 2 != m:
        raise ValueError("bad vech length")
    return d


# --------------------------------------------------------------------------- LSCV_h (Sec 4.4.2)
def lscv_h_scores(X, hs, threads: int = 1, parts: bool = False):
    """g(h) of Eq. 24 for each h: Sigma per Eq. 20-23, det and inverse (steps 2-3),
    T(u) = (K*K)(u) - 2K(u) with u = (X_i-X_j)/h, R(K) = (4pi)^{-d/2}|Sigma|^{-1/2} (reading Z2).
    With parts=True also returns (sum (K*K), sum K) per h for the pins."""
    X = _as_X(X)
    d, n = X.shape
    _, S = mean_cov(X)
    Sinv, det = gauss_jordan(S)
    if Sinv is None or not det > 0.0:
        raise ValueError("singular covariance")
    Sinv = np.ascontiguousarray(Sinv)
    c4 = (4.0 * math.pi) ** (-d / 2.0) * det ** -0.5
    c2 = (2.0 * math.pi) ** (-d / 2.0) * det ** -0.5
    RK = c4
    L = lib()
    out, prt = [], []
    for h in np.asarray(hs, float).ravel():
        if not h > 0.0:
            raise ValueError("h must be > 0")

        def fn(i0, i1, h=h):
            o = np.zeros(2)
            _check(L.oracle_lscv_h_pairsums_rows(_dp(X), n, d, _dp(Sinv), float(h), i0, i1,
                                                 _dp(o)), "lscv_h sums")
            return o

        ea, eb = _parallel_rows(fn, n, threads, 2)
        sumKK, sumK = c4 * ea, c2 * eb
        sumT = sumKK - 2.0 * sumK
        out.append(h ** (-d) * (2.0 * sumT / (n * n) + RK / n))
        prt.append((sumKK, sumK))
    out = np.array(out)
    return (out, np.array(prt)) if parts else out


def lscv_h_modified(X, hs):
    """Sec. 4.5 route (Eq. 36-41): precomputed S(v) buffer, then per-h sums (small n only)."""
    X = _as_X(X)
    d, n = X.shape
    _, S = mean_cov(X)
    Sinv, det = gauss_jordan(S)
    hs = np.ascontiguousarray(np.asarray(hs, float).ravel())
    g = np.zeros(hs.size)
    Sinv = np.ascontiguousarray(Sinv)
    _check(lib().oracle_lscv_h_modified(_dp(X), n, d, _dp(Sinv), det, _dp(hs), hs.size, _dp(g)),
           "lscv_h_modified")
    return g


def lscv_h0(n: int, d: int) -> float:
    """Eq. 25 as written: R(K)/mu2^2 = 1/(2^d pi^{d/2} d^2),
    R(f'') = d(d+2)/(2^{d+2} pi^{d/2}); h0 = (R(K)/(mu2^2 R(f'') n))^{1/(d+4)} (reading Z3)."""
    ratio = 1.0 / (2.0 ** d * math.pi ** (d / 2.0) * d * d)
    Rf2 = d * (d + 2) / (2.0 ** (d + 2) * math.pi ** (d / 2.0))
    return (ratio / (Rf2 * n)) ** (1.0 / (d + 4))


def lscv_h_grid(n: int, d: int, n_grid: int = 150, range_factor: float = 4.0):
    """Z(h0) = [h0/4, 4h0] (Eq. 27) sampled at n_grid linearly spaced points, both
    endpoints included (reading Z4)."""
    h0 = lscv_h0(n, d)
    lo, hi = h0 / range_factor, h0 * range_factor
    return np.array([lo + k * (hi - lo) / (n_grid - 1) for k in range(n_grid)])


def lscv_h_select(X, n_grid: int = 150, range_factor: float = 4.0, threads: int = 1,
                  refine_steps: int = 0, refine_tol: float = 1e-9):
    """argmin over the grid (Eq. 28), ties -> smaller h (reading Z5).  With refine_steps > 0 the
    bracket formed by the argmin's grid neighbours is re-sectioned refine_steps times with 16
    equally spaced interior points each (a batched section search, "Golden ratio")."""
    X = _as_X(X)
    d, n = X.shape
    hs = lscv_h_grid(n, d, n_grid, range_factor)
    g = lscv_h_scores(X, hs, threads)
    k = int(np.argmin(g))          # first minimum = smallest h among ties
    out = dict(h=float(hs[k]), index=k, grid=hs, scores=g, objective=float(g[k]), steps=0)
    if refine_steps > 0:
        pts = [(hs[max(k - 1, 0)], g[max(k - 1, 0)])]
        if k > 0:
            pts.append((hs[k], g[k]))
        if k + 1 < n_grid:
            pts.append((hs[k + 1], g[k + 1]))
        steps = 0
        while steps < refine_steps:
            a, b = pts[0][0], pts[-1][0]
            if not (b - a > refine_tol * out["h"]):
                break
            hh = [a + (i + 1) * (b - a) / 17.0 for i in range(16)]
            gg = lscv_h_scores(X, hh, threads)
            pts = sorted(pts + list(zip(hh, gg)))
            bi = min(range(len(pts)), key=lambda i: (pts[i][1], i))
            out["h"], out["objective"] = float(pts[bi][0]), float(pts[bi][1])
            pts = pts[max(bi - 1, 0): min(bi + 2, len(pts))]
            steps += 1
        out["steps"] = steps
    return out


# --------------------------------------------------------------------------- LSCV_H (Sec 4.4.3)
def lscv_H_score(X, H, threads: int = 1, penalty: float = PENALTY, parts: bool = False):
    """g(H) of Eq. 30-34.  Non-PD H -> penalty (reading Z8)."""
    X = _as_X(X)
    d, n = X.shape
    H = np.asarray(H, float)
    if H.ndim == 1:
        H = unvech(H, d)
    if cholesky_pd(H) is None:
        return (penalty, (np.nan, np.nan)) if parts else penalty
    Hinv, det = gauss_jordan(H)
    Hinv = np.ascontiguousarray(Hinv)
    L = lib()

    def fn(i0, i1):
        o = np.zeros(2)
        _check(L.oracle_lscv_H_pairsums_rows(_dp(X), n, d, _dp(Hinv), i0, i1, _dp(o)),
               "lscv_H sums")
        return o

    ea, eb = _parallel_rows(fn, n, threads, 2)
    c4 = (4.0 * math.pi) ** (-d / 2.0) * det ** -0.5       # (K*K)_H constant, Eq. 33
    c2 = (2.0 * math.pi) ** (-d / 2.0) * det ** -0.5       # K_H constant, Eq. 32
    sumT = c4 * ea - 2.0 * (c2 * eb)                       # Eq. 31
    RK = 2.0 ** (-d) * math.pi ** (-d / 2.0) * det ** -0.5  # Eq. 34
    g = 2.0 * sumT / (n * n) + RK / n                       # Eq. 30
    return (g, (c4 * ea, c2 * eb)) if parts else g


def H_start(X):
    """Eq. 35 as written: (4/(d+2))^{1/(d+4)} n^{-1/(d+4)} Sigma^{1/2}."""
    X = _as_X(X)
    d, n = X.shape
    _, S = mean_cov(X)
    return (4.0 / (d + 2)) ** (1.0 / (d + 4)) * n ** (-1.0 / (d + 4)) * sqrtm_spd(S)


def initial_simplex(x0, d: int):
    """NM start (reading Z8): vertex k = x0 + delta_k e_k, delta = 0.1*H_aa on a diagonal entry
    and 0.1*sqrt(H_aa H_bb) on an off-diagonal entry (a >= b)."""
    H = unvech(x0, d)
    sim = [np.array(x0, float)]
    t = 0
    for b in range(d):
        for a in range(b, d):
            delta = 0.1 * (H[a, a] if a == b else math.sqrt(H[a, a] * H[b, b]))
            v = np.array(x0, float)
            v[t] += delta
            sim.append(v)
            t += 1
    return sim


def nelder_mead(f, sim, max_iter: int = 500, tol: float = 1e-7, trace=None):
    """Standard Nelder–Mead (rho=1, chi=2, gamma=0.5, sigma=0.5), reading Z8 / SURVEY NM spec:
    stable order by (f, vertex index); reflect; expand if f_r < f_1 (accept x_e if f_e < f_r);
    accept x_r if f_1 <= f_r < f_m; outside contraction if f_m <= f_r < f_{m+1} (accept if
    f_c <= f_r); inside contraction if f_r >= f_{m+1} (accept if f_cc < f_{m+1}); otherwise
    shrink toward the best vertex.  Stop when f_{m+1} - f_1 <= tol*|f_1| or after max_iter
    iterations.  `trace`, if a list, receives every (x, f) evaluated in order."""
    sim = [np.array(v, float) for v in sim]
    m = len(sim) - 1

    def ev(x):
        v = f(x)
        if trace is not None:
            trace.append((np.array(x), v))
        return v

    fs = [ev(v) for v in sim]
    it = 0
    stop = "max_iter"
    while True:
        order = sorted(range(m + 1), key=lambda k: (fs[k], k))
        sim = [sim[k] for k in order]
        fs = [fs[k] for k in order]
        if fs[m] - fs[0] <= tol * abs(fs[0]):
            stop = "tol"
            break
        if it >= max_iter:
            break
        it += 1
        xbar = np.add.reduce(sim[:m], 0) / m
        xr = xbar + 1.0 * (xbar - sim[m])
        fr = ev(xr)
        if fr < fs[0]:
            xe = xbar + 2.0 * (xr - xbar)
            fe = ev(xe)
            sim[m], fs[m] = (xe, fe) if fe < fr else (xr, fr)
            continue
        if fr < fs[m - 1]:
            sim[m], fs[m] = xr, fr
            continue
        if fr < fs[m]:
            xc = xbar + 0.5 * (xr - xbar)
            fc = ev(xc)
            if fc <= fr:
                sim[m], fs[m] = xc, fc
                continue
        else:
            xcc = xbar + 0.5 * (sim[m] - xbar)
            fcc = ev(xcc)
            if fcc < fs[m]:
                sim[m], fs[m] = xcc, fcc
                continue
        for k in range(1, m + 1):
            sim[k] = sim[0] + 0.5 * (sim[k] - sim[0])
            fs[k] = ev(sim[k])
    return dict(x=sim[0], f=fs[0], iterations=it, stop=stop, simplex=sim, fvals=fs)


def vech_llt(x, d: int):
    """vech(L L^T) for x = vech(L), L lower triangular (the Cholesky-factor search variables, row f4)."""
    L = np.tril(unvech(x, d))
    return vech(L @ L.T)


def lscv_H_select(X, max_iter: int = 500, tol: float = 1e-7, penalty: float = PENALTY,
                  threads: int = 1, trace=None, nm_starts: int = 1, param: str = "vech"):
    """LSCV_H: minimise g(H) (Eq. 30) over vech(H) by Nelder–Mead from H_start (Eq. 35).
    nm_starts > 1 (row f4): independent runs from the initial simplex scaled by 4^-k, best kept
    (ties -> earlier run).  param = "chol" (row f4): the search variables are vech(L) of a lower
    triangular L with H = L L^T (every vertex positive semi-definite), starting from
    L = chol(H_start); the simplex rule of reading Z8 and the 4^-k scaling apply to L."""
    X = _as_X(X)
    d, n = X.shape
    Hs = H_start(X)
    if param == "chol":
        x0 = vech(cholesky_pd(Hs))
        to_H = lambda v: vech_llt(v, d)
    elif param == "vech":
        x0 = vech(Hs)
        to_H = lambda v: v
    else:
        raise ValueError("param must be 'vech' or 'chol'")
    sim0 = initial_simplex(x0, d)
    best = None
    for k in range(max(1, nm_starts)):
        sim = [v * 4.0 ** (-k) for v in sim0]
        res = nelder_mead(lambda v: lscv_H_score(X, to_H(v), threads, penalty), sim, max_iter, tol, trace)
        if best is None or res["f"] < best["f"]:
            best = res
    best["H"] = unvech(to_H(best["x"]), d)
    best["H_start"] = Hs
    return best


def tile_enumerate(count: int):
    l = np.zeros(count, dtype=np.int64)
    q = np.zeros(count, dtype=np.int64)
    _check(lib().oracle_tile_enumerate(count, l.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                       q.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))), "tiles")
    return l, q


# --------------------------------------------------------------------------- KDE evaluation / AQP
def kde_eval(X, Y, H):
    """fhat(y) for each column y of Y (Eq. kde-def-H / K_H / gaussian).  H is a d x d
    matrix or its vech; the scalar-h estimator of Eq. kde-def is H = h^2 I."""
    X = _as_X(X)
    d, n = X.shape
    Y = np.ascontiguousarray(np.asarray(Y, float).reshape(d, -1))
    m = Y.shape[1]
    H = np.asarray(H, float)
    if H.ndim == 1:
        H = unvech(H, d)
    if cholesky_pd(H) is None:
        raise ValueError("H not positive definite")
    Hinv, det = gauss_jordan(H)
    Hinv = np.ascontiguousarray(Hinv)
    f = np.zeros(m)
    _check(lib().oracle_kde_eval(_dp(X), n, d, _dp(Y), m, _dp(Hinv), det, _dp(f)), "kde_eval")
    return f


def aqp_1d(x, h, a, b, epsrel=1e-12):
    """Approximate COUNT, SUM, AVG of the records with a <= x <= b (Eq. count, sum):
    COUNT = n * integral_a^b fhat(t) dt,  SUM = n * integral_a^b t fhat(t) dt,  AVG = SUM/COUNT,
    fhat the scalar-h Gaussian KDE (Eq. kde-def).  The integrals are done by adaptive
    quadrature (scipy.integrate.quad) of the oracle's own fhat, as the paper allows."""
    import scipy.integrate as si
    x = np.asarray(x, float).ravel()
    n = x.size
    f = lambda t: float(kde_eval(x[None, :], np.array([[t]]), [h * h])[0])
    # split the interval at the sample-dense points to help quad
    pts = np.linspace(a, b, 9)
    cnt = sum(si.quad(f, p0, p1, epsabs=0, epsrel=epsrel, limit=200)[0] for p0, p1 in zip(pts[:-1], pts[1:]))
    sm = sum(si.quad(lambda t: t * f(t), p0, p1, epsabs=1e-300, epsrel=epsrel, limit=200)[0]
             for p0, p1 in zip(pts[:-1], pts[1:]))
    return n * cnt, n * sm, (sm / cnt if cnt != 0 else float("nan"))
