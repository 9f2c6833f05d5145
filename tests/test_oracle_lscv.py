"""Pins for the oracle's LSCV_h / LSCV_H objectives, start rules and Nelder–Mead (CPU only)."""
import math

import numpy as np
import pytest
import scipy.integrate as si
import scipy.linalg as sl
import scipy.optimize as so
import scipy.stats as st

import datagen
import oracle


def _kde_sq_integral_1d(x, H):
    """integral of fhat_H(t)^2 dt for d=1 by quadrature of the KDE built with scipy.stats.norm."""
    s = math.sqrt(H)
    f = lambda t: np.mean(st.norm.pdf(t, loc=x, scale=s)) ** 2
    pts = np.linspace(x.min() - 12 * s, x.max() + 12 * s, 61)
    return sum(si.quad(f, a, b, epsabs=0, epsrel=1e-13, limit=200)[0] for a, b in zip(pts[:-1], pts[1:]))


def test_lscv_H_d1_equals_ise_identity():
    # g(H) = int fhat_H^2 - 4 n^-2 sum_{i<j} K_H(X_i - X_j)  (Eq. 30-34 with the paper's 2n^-2
    # normalisation, reading Z6).  The integral is computed by quadrature of a scipy-built KDE,
    # the K_H sum by scipy's normal pdf: both independent of the oracle's exp formula.
    x = np.array([0.0, 1.0, 1.1, 1.5, 1.9, 2.8, 2.9, 3.5])   # P:163 toy data
    n = x.size
    for H in [0.05, 0.3, 1.2]:
        ise = _kde_sq_integral_1d(x, H)
        sK = sum(st.norm.pdf(x[i] - x[j], scale=math.sqrt(H)) for i in range(n) for j in range(i + 1, n))
        g = oracle.lscv_H_score(x[None, :], [H])
        assert g == pytest.approx(ise - 4 * sK / n ** 2, rel=1e-10)


def test_lscv_H_d2_parts_match_scipy_mvn_and_ise():
    X = datagen.sample_mixture("C3", 6, 3)
    n = X.shape[1]
    H = np.array([[0.3, 0.08], [0.08, 0.2]])
    g, (sKK, sK) = oracle.lscv_H_score(X, H, parts=True)
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    d = X[:, [i for i, _ in pairs]] - X[:, [j for _, j in pairs]]
    assert sK == pytest.approx(st.multivariate_normal(cov=H).pdf(d.T).sum(), rel=1e-12)          # K_H = N(0,H)
    assert sKK == pytest.approx(st.multivariate_normal(cov=2 * H).pdf(d.T).sum(), rel=1e-12)     # (K*K)_H = N(0,2H)
    # ISE identity in 2-D: int fhat^2 by dblquad
    mv = st.multivariate_normal(cov=H)
    f = lambda y, x: np.mean(mv.pdf(np.stack([x - X[0], y - X[1]], -1))) ** 2
    lo, hi = X.min() - 4, X.max() + 4
    ise = si.dblquad(f, lo, hi, lo, hi, epsabs=1e-13, epsrel=1e-10)[0]
    assert g == pytest.approx(ise - 4 * sK / n ** 2, rel=1e-7)


@pytest.mark.parametrize("d,n", [(1, 64), (2, 64), (4, 48)])
def test_modified_equals_unmodified(d, n):
    # Sec. 4.5 claim: Eq. 41 with precomputed S(v) equals Eq. 24.
    X = np.random.default_rng(d).normal(size=(d, n)) @ np.diag(np.linspace(1, 2, n))
    hs = np.linspace(0.1, 2.0, 20)
    a = oracle.lscv_h_scores(X, hs)
    b = oracle.lscv_h_modified(X, hs)
    np.testing.assert_allclose(a, b, rtol=1e-12)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_cross_selector_identity(d):
    # The Sigma-shaped scalar-h kernel is K_H with H = h^2 Sigma, so g_h(h) = g_H(h^2 Sigma)
    # exactly (different code routes: u=(Xi-Xj)/h with Sigma^-1 vs (h^2 Sigma)^-1).
    X = datagen.sample_mixture("C5", 40, 8)[:d] if d > 1 else datagen.sample_mixture("bimodal", 40, 8)
    _, S = oracle.mean_cov(X)
    for h in [0.2, 0.6, 1.4]:
        gh = oracle.lscv_h_scores(X, [h])[0]
        gH = oracle.lscv_H_score(X, h * h * S)
        assert gh == pytest.approx(gH, rel=1e-12)


def test_n2_special_values():
    # n=2, d=1, X1=X2, H=[1]: g = 0.5 [(4pi)^-1/2 - 2(2pi)^-1/2] + 0.5 (2 sqrt(pi))^-1
    g = oracle.lscv_H_score(np.array([[0.7, 0.7]]), [1.0])
    assert g == pytest.approx(-0.1168474886, abs=1e-10)
    # T~(0) with Sigma=1, h=1: (4pi)^-1/2 - 2 (2pi)^-1/2 = -0.5157897690
    assert (4 * math.pi) ** -0.5 - 2 * (2 * math.pi) ** -0.5 == pytest.approx(-0.5157897690, abs=1e-10)


def test_non_pd_penalty():
    X = datagen.sample_mixture("C3", 20, 3)
    assert oracle.lscv_H_score(X, np.array([[1.0, 2.0], [2.0, 1.0]])) == oracle.PENALTY
    assert oracle.lscv_H_score(X, np.array([[-1.0, 0.0], [0.0, 1.0]])) == oracle.PENALTY


def test_expectation_mixture_lscv():
    # E[g(H)] = n^-1 (4pi)^{-d/2}|H|^{-1/2}
    #          + (1-1/n) sum_lm w_l w_m [phi_{2H+S_l+S_m}(mu_l-mu_m) - 2 phi_{H+S_l+S_m}(mu_l-mu_m)]
    # (exact MISE algebra of normal mixtures).  MC z-test.
    w, mus, covs = datagen.mixture("C3")
    n, seeds = 150, 120
    H = np.array([[0.12, 0.03], [0.03, 0.09]])
    E = (4 * math.pi) ** -1 * np.linalg.det(H) ** -0.5 / n
    for wl, ml, cl in zip(w, mus, covs):
        for wm, mm, cm in zip(w, mus, covs):
            E += (1 - 1 / n) * wl * wm * (st.multivariate_normal(cov=2 * H + cl + cm).pdf(ml - mm)
                                          - 2 * st.multivariate_normal(cov=H + cl + cm).pdf(ml - mm))
    vals = np.array([oracle.lscv_H_score(datagen.sample_mixture("C3", n, s), H) for s in range(500, 500 + seeds)])
    z = (vals.mean() - E) / (vals.std(ddof=1) / math.sqrt(seeds))
    assert abs(z) < 4.0, (vals.mean(), E, z)


def test_h0_and_grid():
    # d=1: Eq. 25 gives the normal-scale h0 = (4/(3n))^{1/5}; n=1000 -> 0.2660649994
    assert oracle.lscv_h0(1000, 1) == pytest.approx(0.2660649994, rel=1e-9)
    assert oracle.lscv_h0(65536, 1) == pytest.approx(0.1152634889, rel=1e-9)
    hs = oracle.lscv_h_grid(1000, 1, 150)
    assert hs.size == 150 and hs[0] == pytest.approx(0.2660649994 / 4) and hs[-1] == pytest.approx(4 * 0.2660649994)


def test_lscv_h_select_argmin_and_ties():
    X = datagen.sample_mixture("bimodal", 300, 2)
    r = oracle.lscv_h_select(X, n_grid=40)
    assert r["scores"][r["index"]] == r["scores"].min()
    assert np.all(r["scores"][: r["index"]] > r["scores"][r["index"]])


def test_matrix_sqrt_and_H_start():
    rng = np.random.default_rng(3)
    A = rng.normal(size=(4, 4))
    S = A @ A.T + 0.3 * np.eye(4)
    np.testing.assert_allclose(oracle.sqrtm_spd(S), np.real(sl.sqrtm(S)), rtol=1e-10, atol=1e-12)
    w, V = oracle.jacobi_eigh(S)
    np.testing.assert_allclose(np.sort(w), np.linalg.eigvalsh(S), rtol=1e-12)
    # d=1, Sigma=1, n=1 -> (4/3)^{1/5} = 1.0592238410; here via equivariance in n:
    X = np.array([[-1.0, 1.0]])   # n=2, Sigma = 2
    Hs = oracle.H_start(X)
    assert Hs[0, 0] == pytest.approx((4 / 3) ** 0.2 * 2 ** -0.2 * math.sqrt(2.0), rel=1e-12)
    assert (4 / 3) ** 0.2 == pytest.approx(1.0592238410, rel=1e-9)


def test_vech_paper_example():
    A = np.array([[1, 4, 7], [2, 5, 8], [3, 6, 9]])
    assert list(oracle.vech(A)) == [1, 2, 3, 5, 6, 9]


def _rosen(x):
    return sum(100.0 * (x[1:] - x[:-1] ** 2) ** 2 + (1 - x[:-1]) ** 2)


def test_nelder_mead_matches_scipy_step_for_step():
    # With the same initial simplex, no ties and a fixed iteration budget, scipy's (non-adaptive)
    # Nelder–Mead makes the same decisions as the spec (rho=1, chi=2, gamma=sigma=0.5); vertex
    # values agree to rounding (scipy writes x_r = 2 xbar - x, we write xbar + (xbar - x)).
    x0 = np.array([-1.2, 1.0, 0.7])
    sim = [x0] + [x0 + 0.1 * e for e in np.eye(3)]
    for iters in (5, 17, 60, 150):
        # scipy counts from 1 and stops at iterations == maxiter: it performs maxiter-1 steps
        ours = oracle.nelder_mead(_rosen, sim, max_iter=iters - 1, tol=0.0)
        ref = so.minimize(_rosen, x0, method="Nelder-Mead",
                          options=dict(initial_simplex=np.array(sim), maxiter=iters, maxfev=10 ** 9,
                                       xatol=0.0, fatol=0.0, adaptive=False))
        np.testing.assert_allclose(np.sort(ours["fvals"]), np.sort(ref.final_simplex[1]), rtol=1e-9)
        np.testing.assert_allclose(ours["x"], ref.final_simplex[0][0], rtol=1e-9)


def test_nelder_mead_finds_quadratic_minimum():
    A = np.array([[3.0, 0.5], [0.5, 1.0]])
    c = np.array([0.3, -0.2])
    f = lambda x: float((x - c) @ A @ (x - c)) + 1.0
    r = oracle.nelder_mead(f, [np.zeros(2), np.array([0.5, 0]), np.array([0, 0.5])], max_iter=500, tol=1e-14)
    np.testing.assert_allclose(r["x"], c, atol=1e-5)
    assert r["stop"] == "tol"


def test_lscv_H_select_small():
    X = datagen.sample_mixture("C3", 120, 7)
    r = oracle.lscv_H_select(X, max_iter=300)
    assert oracle.cholesky_pd(r["H"]) is not None
    assert r["f"] <= oracle.lscv_H_score(X, r["H_start"])
    # d=1 consistency with a dense scalar scan: optimum H ~ h*^2 within 5% on h
    x = datagen.sample_mixture("bimodal", 150, 5)
    r1 = oracle.lscv_H_select(x, max_iter=300, tol=1e-10)
    hs = np.linspace(0.02, 1.5, 400)
    gs = [oracle.lscv_H_score(x, [h * h]) for h in hs]
    hstar = hs[int(np.argmin(gs))]
    assert math.sqrt(r1["H"][0, 0]) == pytest.approx(hstar, rel=0.05)


def test_lscv_h_refinement_finds_continuous_minimum():
    # The refined LSCV_h argmin agrees with a bounded scalar minimiser on the same objective
    # (scipy.optimize.minimize_scalar) inside the grid bracket (f4 row).
    X = datagen.sample_mixture("bimodal", 400, 12)
    r = oracle.lscv_h_select(X, n_grid=40, refine_steps=8, refine_tol=1e-10)
    k = r["index"]
    lo, hi = r["grid"][max(k - 1, 0)], r["grid"][min(k + 1, 39)]
    ref = so.minimize_scalar(lambda h: oracle.lscv_h_scores(X, [h])[0], bounds=(lo, hi), method="bounded",
                             options=dict(xatol=1e-12))
    assert r["h"] == pytest.approx(ref.x, rel=1e-6)
    assert r["objective"] <= ref.fun + 1e-15


def test_mean_cov_matches_numpy():
    # Eq. 20-23 (unbiased sample covariance, reading Z10) vs numpy's library routine
    X = datagen.sample_mixture("C5", 500, 3)
    m, S = oracle.mean_cov(X)
    np.testing.assert_allclose(m, X.mean(axis=1), rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(S, np.cov(X), rtol=1e-12, atol=1e-15)
    # Eq. 11 one-pass form equals the two-pass value for well-scaled data
    x = X[0]
    n = x.size
    V11 = (x ** 2).sum() / (n - 1) - x.sum() ** 2 / (n * (n - 1))
    assert S[0, 0] == pytest.approx(V11, rel=1e-12)


def test_vech_llt_hand_example():
    # L = [[2, 0], [1, 3]]: vech(L) = [2, 1, 3] (P:351-363 order), L L^T = [[4, 2], [2, 10]]
    np.testing.assert_array_equal(oracle.vech_llt([2.0, 1.0, 3.0], 2), [4.0, 2.0, 10.0])
    # d = 3, checked against numpy's product of the unpacked factor
    x = np.array([1.5, -0.5, 0.25, 2.0, 0.75, 0.5])
    L = np.array([[1.5, 0, 0], [-0.5, 2.0, 0], [0.25, 0.75, 0.5]])
    H = L @ L.T
    np.testing.assert_allclose(oracle.vech_llt(x, 3), [H[0, 0], H[1, 0], H[2, 0], H[1, 1], H[2, 1], H[2, 2]], rtol=1e-15)


def test_lscv_H_select_cholesky_parametrisation():
    # Row f4 variant: the search over vech(L), H = L L^T.  d = 1 pins it to a dense scalar scan of the
    # same objective (the optimum L^2 = h*^2, within the scan and tolerance resolution), and at d = 2
    # it reaches an objective no worse than the vech(H) search's within the NM tolerance band.
    x = datagen.sample_mixture("bimodal", 150, 5)
    r = oracle.lscv_H_select(x, max_iter=300, tol=1e-10, param="chol")
    hs = np.linspace(0.02, 1.5, 400)
    gs = [oracle.lscv_H_score(x, [h * h]) for h in hs]
    assert math.sqrt(r["H"][0, 0]) == pytest.approx(hs[int(np.argmin(gs))], rel=0.05)
    assert r["f"] == pytest.approx(oracle.lscv_H_score(x, [r["H"][0, 0]]), rel=1e-15)
    X = datagen.sample_mixture("C3", 200, 9)
    rc = oracle.lscv_H_select(X, max_iter=400, param="chol")
    rv = oracle.lscv_H_select(X, max_iter=400)
    assert oracle.cholesky_pd(rc["H"]) is not None
    assert rc["f"] <= rv["f"] + 1e-4 * abs(rv["f"])
    # the start: L = chol(H_start), so the first vertex is H_start itself
    L0 = oracle.cholesky_pd(rc["H_start"])
    np.testing.assert_allclose(oracle.vech_llt(oracle.vech(L0), 2), oracle.vech(rc["H_start"]), rtol=1e-14)
