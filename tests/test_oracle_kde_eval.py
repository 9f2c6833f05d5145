"""Pins for the oracle's KDE evaluation and AQP aggregates, CPU only."""
import math

import numpy as np
import pytest
import scipy.integrate as si
import scipy.special as ss
import scipy.stats as st

import datagen
import oracle


def test_kde_eval_matches_scipy_mvn_sum():
    # fhat(y) = n^-1 sum_i N(y; X_i, H)  (Eq. kde-def-H with K_H)
    X = datagen.sample_mixture("C3", 40, 5)
    Y = datagen.sample_mixture("C3", 7, 6)
    H = np.array([[0.2, 0.05], [0.05, 0.15]])
    f = oracle.kde_eval(X, Y, H)
    ref = [np.mean(st.multivariate_normal(mean=Y[:, q], cov=H).pdf(X.T)) for q in range(Y.shape[1])]
    np.testing.assert_allclose(f, ref, rtol=1e-13)


def test_kde_scalar_h_is_H_h2_identity():
    # Eq. kde-def (scalar h, K_h) equals Eq. kde-def-H with H = h^2 I; scipy's gaussian_kde
    # with a fixed factor on unit-covariance data is the same estimator.
    x = np.array([0.0, 1.0, 1.1, 1.5, 1.9, 2.8, 2.9, 3.5])
    h = 0.4
    y = np.linspace(-1, 4.5, 23)
    f = oracle.kde_eval(x[None, :], y[None, :], [h * h])
    ref = [np.mean(st.norm.pdf(t, loc=x, scale=h)) for t in y]
    np.testing.assert_allclose(f, ref, rtol=1e-13)


def test_kde_integrates_to_one():
    x = datagen.sample_mixture("skewed", 30, 2)
    tot = si.quad(lambda t: oracle.kde_eval(x, np.array([[t]]), [0.09])[0], -20, 20, limit=400, epsabs=1e-13)[0]
    assert tot == pytest.approx(1.0, abs=1e-10)


def test_aqp_quadrature_matches_closed_form():
    # COUNT = sum_i [Phi(beta_i) - Phi(alpha_i)], SUM adds h (phi(alpha_i) - phi(beta_i)) + x_i (...)
    # (closed forms of Eq. count / Eq. sum for the Gaussian kernel) via scipy.special.ndtr.
    x = datagen.sample_mixture("bimodal", 50, 3)[0]
    h = 0.3
    for a, b in [(-1.0, 0.5), (0.2, 2.0), (-5.0, 5.0)]:
        cnt, sm, avg = oracle.aqp_1d(x, h, a, b)
        al, be = (a - x) / h, (b - x) / h
        c_ref = np.sum(ss.ndtr(be) - ss.ndtr(al))
        s_ref = np.sum(x * (ss.ndtr(be) - ss.ndtr(al)) + h * (st.norm.pdf(al) - st.norm.pdf(be)))
        assert cnt == pytest.approx(c_ref, rel=1e-10)
        assert sm == pytest.approx(s_ref, rel=1e-9, abs=1e-9)
        assert avg == pytest.approx(s_ref / c_ref, rel=1e-9)


def test_aqp_whole_line_counts_everything():
    x = datagen.sample_mixture("N01", 40, 8)[0]
    cnt, sm, avg = oracle.aqp_1d(x, 0.25, -40.0, 40.0)
    assert cnt == pytest.approx(x.size, rel=1e-10)
    assert sm == pytest.approx(x.sum(), rel=1e-9, abs=1e-9)
