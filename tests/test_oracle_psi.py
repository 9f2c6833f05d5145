"""Pins for the oracle's Psi_r-hat sums and PLUGIN chain (CPU only).

Every check compares the oracle with something other than itself: symbolic differentiation
(sympy), library Hermite polynomials + numerical quadrature (scipy), closed forms from the
normal-reference theory, Monte-Carlo expectations, and exact invariances.
"""
import math

import numpy as np
import pytest
import scipy.integrate as si
import scipy.special as ss
import sympy as sp

import datagen
import oracle

TOY = np.array([0.0, 1.0, 1.1, 1.5, 1.9, 2.8, 2.9, 3.5])   # PAPER.md P:163 (Fig. 1 toy data)


def phi_deriv(k, x, s):
    """k-th derivative of the N(0, s^2) density, via scipy's He_k (library routine)."""
    z = x / s
    return (-1) ** k * ss.eval_hermitenorm(k, z) * np.exp(-0.5 * z * z) / (math.sqrt(2 * math.pi) * s ** (k + 1))


@pytest.mark.parametrize("r", [4, 6, 8])
def test_kernel_derivative_matches_sympy(r):
    # K^(r) = d^r/du^r of the Gaussian kernel: symbolic differentiation pins the
    # Hermite coefficients (a dropped term or wrong sign fails here).
    u = sp.symbols("u")
    dr = sp.lambdify(u, sp.diff(sp.exp(-u ** 2 / 2) / sp.sqrt(2 * sp.pi), u, r), "math")
    for val in [0.0, 0.3, -0.7, 1.0, 1.9, 2.5, -3.3, 5.0]:
        assert oracle.kernel_deriv(r, val) == pytest.approx(dr(val), rel=1e-12, abs=1e-15)


def test_kernel_constants_at_zero():
    # P:222 K^6(0) = -15/sqrt(2pi); P:238 K^4(0) = 3/sqrt(2pi); He_8(0) = 105 = 7!!.
    s2p = math.sqrt(2 * math.pi)
    assert oracle.kernel_deriv(6, 0.0) == pytest.approx(-15 / s2p, rel=1e-15)
    assert oracle.kernel_deriv(4, 0.0) == pytest.approx(3 / s2p, rel=1e-15)
    assert oracle.hermite(8, 0.0) == 105.0


@pytest.mark.parametrize("r", [4, 6, 8])
@pytest.mark.parametrize("g", [0.3, 0.7, 1.6])
def test_psi_equals_quadrature_identity(r, g):
    # With the diagonal included, sum_i sum_j phi_g^(r)(X_i-X_j)
    #   = (-1)^{r/2} * integral( (sum_i phi_{g/sqrt2}^{(r/2)}(x - X_i))^2 dx ),
    # and n^2 Psi_r-hat(g) equals the left side (reading Z1).  The right side uses only
    # He_{r/2} from scipy and numerical quadrature: independent of the oracle's He_r.
    x = TOY
    n = x.size
    s = g / math.sqrt(2.0)
    k = r // 2

    def f2(t):
        return np.sum(phi_deriv(k, t - x, s)) ** 2

    lo, hi = x.min() - 12 * s, x.max() + 12 * s
    pts = list(np.linspace(lo, hi, 41))
    val = sum(si.quad(f2, a, b, epsabs=0, epsrel=1e-13, limit=200)[0] for a, b in zip(pts[:-1], pts[1:]))
    rhs = (-1) ** k * val / (n * n)
    assert oracle.psi_r(x, r, g) == pytest.approx(rhs, rel=1e-9)


def test_sign_theorem_random_and_adversarial():
    # sign(Psi_r-hat) = (-1)^{r/2} always (consequence of the identity above, reading Z11).
    rng = np.random.default_rng(11)
    cases = [rng.normal(size=rng.integers(2, 40)) for _ in range(30)]
    cases += [np.array([0.0, 0.0, 0.0, 5.0]), np.array([0.0, 100.0]), np.r_[np.zeros(10), 1e-3]]
    for x in cases:
        for g in [0.01, 0.2, 1.0, 10.0]:
            for r in (4, 6, 8):
                v = oracle.psi_r(x, r, g)
                assert (v > 0) == (r % 4 == 0), (r, g, x)


@pytest.mark.parametrize("r", [4, 6, 8])
def test_psi_ns_closed_form_matches_quadrature(r):
    # Normal-reference functional Psi_r^NS(sigma) = (-1)^{r/2} int (f^{(r/2)})^2 for f=N(0,s^2),
    # closed form (-1)^{r/2} r!/((2s)^{r+1} (r/2)! sqrt(pi)) (BASELINE.json north_star).
    sig = 1.3
    val = si.quad(lambda t: phi_deriv(r // 2, t, sig) ** 2, -30, 30, epsabs=0, epsrel=1e-13, limit=400)[0]
    closed = (-1) ** (r // 2) * math.factorial(r) / ((2 * sig) ** (r + 1) * math.factorial(r // 2) * math.sqrt(math.pi))
    assert (-1) ** (r // 2) * val == pytest.approx(closed, rel=1e-10)
    if r == 8:  # the PLUGIN step-3 constant (Eq. 13)
        x = datagen.sample_mixture("N01", 50, 9)[0]
        t = oracle.plugin(x)
        s = t["sigma_hat"]
        v8 = si.quad(lambda z: phi_deriv(4, z, s) ** 2, -40 * s, 40 * s, epsabs=0, epsrel=1e-13, limit=400)[0]
        assert t["psi8_ns"] == pytest.approx(v8, rel=1e-9)


def test_worked_example_x123():
    # X=[1,2,3]: V=1, sigma=1 exactly (Eq. 11-12); Psi8NS = 105/(32 sqrt(pi)) = Psi_8^NS(1).
    # (SPEC S:338 prints 1.85056 — an erratum; the closed form gives 1.851247071016...)
    t = oracle.plugin([1.0, 2.0, 3.0])
    assert t["V_hat"] == 1.0 and t["sigma_hat"] == 1.0
    assert t["psi8_ns"] == pytest.approx(105 / (32 * math.sqrt(math.pi)), rel=1e-15)
    # n=2-style closed check of the Psi_6 bracket: pairs (1,2),(1,3),(2,3) have |d| = 1,2,1.
    g = t["g1"]
    K6 = lambda u: float(sp.diff(sp.exp(-sp.Symbol("u") ** 2 / 2) / sp.sqrt(2 * sp.pi), sp.Symbol("u"), 6).subs(sp.Symbol("u"), u))
    S = 2 * K6(1 / g) + K6(2 / g)
    assert t["psi6"] == pytest.approx((2 * S + 3 * K6(0)) / (9 * g ** 7), rel=1e-12)


def test_expectation_normal_data():
    # E[Psi_r-hat(g)] = g^{-r-1} K^(r)(0)/n + (1-1/n) Psi_r^NS(sqrt(sigma^2 + g^2/2)) for
    # N(0, sigma^2) data (SURVEY §8(c) pins table; from E phi_g^(r)(X-Y) = phi^(r)_{sqrt(g^2+2s^2)}(0)).
    n, seeds = 400, 48
    for r, g in [(4, 0.5), (6, 0.4), (8, 0.6)]:
        vals = np.array([oracle.psi_r(datagen.sample_mixture("N01", n, s)[0], r, g) for s in range(100, 100 + seeds)])
        sp_ = math.sqrt(1 + g * g / 2)
        ns = (-1) ** (r // 2) * math.factorial(r) / ((2 * sp_) ** (r + 1) * math.factorial(r // 2) * math.sqrt(math.pi))
        K0 = ss.eval_hermitenorm(r, 0) / math.sqrt(2 * math.pi)
        E = K0 / (n * g ** (r + 1)) + (1 - 1 / n) * ns
        z = (vals.mean() - E) / (vals.std(ddof=1) / math.sqrt(seeds))
        assert abs(z) < 4.0, (r, g, vals.mean(), E, z)


def test_expectation_mixture_data():
    # Mixture generalisation: E[phi_g^(r)(X-Y)] = sum_lm w_l w_m phi^(r)_{sqrt(g^2+s_l^2+s_m^2)}(mu_l-mu_m)
    w, mus, covs = datagen.mixture("skewed")
    n, seeds, r, g = 300, 48, 6, 0.3
    E_off = 0.0
    for wl, ml, cl in zip(w, mus, covs):
        for wm, mm, cm in zip(w, mus, covs):
            s = math.sqrt(g * g + cl[0, 0] + cm[0, 0])
            E_off += wl * wm * phi_deriv(r, float(ml[0] - mm[0]), s)
    K0 = ss.eval_hermitenorm(r, 0) / math.sqrt(2 * math.pi)
    E = K0 / (n * g ** (r + 1)) + (1 - 1 / n) * E_off
    vals = np.array([oracle.psi_r(datagen.sample_mixture("skewed", n, s)[0], r, g) for s in range(300, 300 + seeds)])
    z = (vals.mean() - E) / (vals.std(ddof=1) / math.sqrt(seeds))
    assert abs(z) < 4.0, (vals.mean(), E, z)


def test_invariances():
    x = datagen.sample_mixture("skewed", 200, 3)[0]
    rng = np.random.default_rng(5)
    for r in (4, 6, 8):
        g = 0.37
        base = oracle.psi_r(x, r, g)
        assert oracle.psi_r(x + 12.5, r, g) == pytest.approx(base, rel=1e-10)          # translation
        assert oracle.psi_r(rng.permutation(x), r, g) == pytest.approx(base, rel=1e-12)  # permutation
        c = 3.7                                                                          # scale
        assert oracle.psi_r(c * x, r, c * g) == pytest.approx(c ** -(r + 1) * base, rel=1e-11)
    h = oracle.plugin(x)["h"]
    assert oracle.plugin(3.7 * x)["h"] == pytest.approx(3.7 * h, rel=1e-10)


def test_pair_symmetry_full_square():
    # Full double sum over all (i,j) = 2 * upper triangle + n K(0) (P:539-552 tiling of the
    # upper triangle only).
    x = datagen.sample_mixture("N01", 60, 4)[0]
    g = 0.5
    for r in (4, 6, 8):
        full = sum(oracle.kernel_deriv(r, (a - b) / g) for a in x for b in x)
        up = oracle.psi_pairsum(x, r, g)
        assert full == pytest.approx(2 * up + x.size * oracle.kernel_deriv(r, 0.0), rel=1e-11, abs=1e-9)


def test_plugin_normal_reference_limit():
    # For N(0,1) data the PLUGIN h approaches the AMISE-optimal h = (R(K)/(mu2^2 R(f'') n))^{1/5};
    # R(f'') by quadrature (independent of the chain's constants).
    n = 1000
    Rf2 = si.quad(lambda t: phi_deriv(2, t, 1.0) ** 2, -30, 30, epsabs=0, epsrel=1e-12)[0]
    h_amise = (1 / (2 * math.sqrt(math.pi)) / (Rf2 * n)) ** 0.2
    hs = [oracle.plugin(datagen.sample_mixture("N01", n, s)[0]) for s in range(1, 17)]
    ratio = np.mean([t["h"] / t["sigma_hat"] for t in hs])
    assert abs(ratio / h_amise - 1) < 0.03
    # rate: h(16384)/h(1024) ~ 16^{-1/5} (SPEC S:388 invariants), median of 3 seeds
    r = [oracle.plugin(datagen.sample_mixture("N01", 4096, s)[0])["h"] / oracle.plugin(datagen.sample_mixture("N01", 256, s)[0])["h"] for s in (1, 2, 3)]
    assert 0.85 < np.median(r) / 16 ** -0.2 < 1.15


def test_plugin_degenerate_and_errors():
    with pytest.raises(oracle.DegenerateData):
        oracle.plugin([2.0, 2.0, 2.0])
    with pytest.raises(ValueError):
        oracle.plugin([1.0])


def test_row_split_parts_add_up():
    x = datagen.sample_mixture("bimodal", 500, 2)[0]
    full = oracle.psi_pairsum(x, 6, 0.2)
    par = oracle.psi_pairsum(x, 6, 0.2, threads=4)
    assert par == pytest.approx(full, rel=1e-13)
    parts = sum(oracle.psi_pairsum(x, 6, 0.2, rows=c) for c in oracle.row_chunks(500, 7))
    assert parts == pytest.approx(full, rel=1e-13)


def test_tile_enumeration_is_column_major_upper_triangle():
    l, q = oracle.tile_enumerate(10_000)
    assert l[0] == 0 and q[0] == 0 and (l[2], q[2]) == (1, 1) and (l[5], q[5]) == (2, 2)
    assert np.all(q <= l)
    assert len(set(zip(l.tolist(), q.tolist()))) == 10_000
