"""GPU parity for KDE evaluation and AQP against the fp64 oracle."""
import numpy as np
import pytest

import datagen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1505_01998_b200 as kb  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = kb.Context()
    yield c
    c.close()


def _H(d, seed, scale):
    A = np.random.default_rng(seed).normal(size=(d, d))
    return scale * (A @ A.T / d + 0.4 * np.eye(d))


@pytest.mark.parametrize("d,n,m", [(1, 1, 1), (1, 5, 3), (1, 1023, 511), (1, 1025, 513), (1, 5000, 2000),
                                   (2, 3000, 700), (3, 1500, 512), (4, 2049, 300), (7, 800, 100), (16, 300, 50)])
def test_evaluate_matches_oracle(ctx, d, n, m):
    if d <= 4:
        X = datagen.sample_mixture("C5", n, 3 + n)[:d]
        Y = datagen.sample_mixture("C5", m, 4 + m)[:d] * 1.3
    else:
        X = np.random.default_rng(n).normal(size=(d, n))
        Y = np.random.default_rng(m).normal(size=(d, m))
    H = _H(d, d, 0.15)
    got = ctx.evaluate(kb.to_device(X), kb.to_device(Y), H)
    ref = oracle.kde_eval(X, Y, H)
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-12 * ref.max())


def test_evaluate_far_queries_and_errors(ctx):
    x = datagen.sample_mixture("N01", 1000, 2)
    y = np.array([[0.0, 40.0, -1e3]])
    got = ctx.evaluate(kb.to_device(x), kb.to_device(y), [0.09])
    ref = oracle.kde_eval(x, y, [0.09])
    assert abs(got[0] - ref[0]) <= 1e-5 * ref[0] and got[1] == 0.0 and got[2] == 0.0
    with pytest.raises(kb.KDEError) as e:
        ctx.evaluate(kb.to_device(x), kb.to_device(y), [-1.0])
    assert e.value.status == "KDE_E_NONPOSITIVE_BW"


def test_aqp_matches_oracle(ctx):
    x = datagen.config_data("C2", n=3000)
    h = 0.12
    lo = np.array([-1.0, 0.0, -3.0, 0.5, 2.0])
    hi = np.array([0.5, 0.0, 3.0, 0.51, 9.0])
    cnt, sm, avg = ctx.aqp_1d(kb.to_device(x), h, lo, hi)
    for q in range(lo.size):
        c, s, a = oracle.aqp_1d(x[0], h, lo[q], hi[q])
        assert cnt[q] == pytest.approx(c, rel=1e-9, abs=1e-12)
        assert sm[q] == pytest.approx(s, rel=1e-8, abs=1e-9)
        if c > 1e-9:
            assert avg[q] == pytest.approx(a, rel=1e-8)


@pytest.mark.parametrize("d", [1, 2])
def test_evaluate_sorted_skip_path_unsorted_queries(ctx, d):
    # >= 2^32 pairs: samples and queries are sorted by coordinate 0, far sample tiles skipped (DESIGN
    # §3.11) and the results scattered back to the caller's query order; 64 random queries (tails
    # included) against the fp64 oracle, same tolerance as above.
    n, m = 1 << 17, 1 << 15
    X = datagen.sample_mixture("C5", n, 31)[:d]
    Y = datagen.sample_mixture("C5", m, 32)[:d] * 1.6          # unsorted, some far in the tails
    H = _H(d, 5, 0.02)
    got = ctx.evaluate(kb.to_device(X), kb.to_device(Y), H)
    idx = np.random.default_rng(7).choice(m, 64, replace=False)
    ref = oracle.kde_eval(X, Y[:, idx], H)
    peak = oracle.kde_eval(X, X[:, :256], H).max()
    np.testing.assert_allclose(got[idx], ref, rtol=1e-5, atol=1e-12 * peak)
