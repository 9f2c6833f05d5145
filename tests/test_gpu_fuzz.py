"""Seeded randomized parity sweep (GPU vs oracle) over sizes around every tile edge (256, 512,
1024, 2048), dimensions and bandwidth scales, for each kernel family."""
import numpy as np
import pytest

import datagen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1505_01998_b200 as kb  # noqa: E402

RNG = np.random.default_rng(20261017)
EDGES = [2, 3, 4, 5, 7, 255, 256, 257, 511, 512, 513, 1023, 1024, 1025, 2047, 2048, 2049]
CASES = [(int(n), int(RNG.integers(1, 5)), float(10 ** RNG.uniform(-1.3, 0.3))) for n in EDGES] + \
        [(int(RNG.integers(2, 3000)), int(RNG.integers(1, 7)), float(10 ** RNG.uniform(-1.3, 0.3))) for _ in range(12)]


@pytest.fixture(scope="module")
def ctx():
    c = kb.Context()
    yield c
    c.close()


def _data(n, d, seed):
    r = np.random.default_rng(seed)
    A = r.normal(size=(d, d)) / np.sqrt(d) + np.eye(d)
    X = A @ r.standard_t(5, size=(d, n))          # heavy-ish tails
    return X + r.normal(size=(d, 1)) * 3          # off-centre


@pytest.mark.parametrize("n,d,scale", CASES)
def test_fuzz_parity(ctx, n, d, scale):
    X = _data(n, d, n * 31 + d)
    Xd = kb.to_device(X)
    # Psi_r (d = 1 view of the first coordinate)
    x1 = np.ascontiguousarray(X[:1])
    g = scale * max(np.std(x1), 1e-3)
    for r in (4, 6, 8):
        got = ctx.psi_r(kb.to_device(x1), r, [g])[0]
        ref = oracle.psi_r(x1[0], r, g)
        assert abs(got - ref) <= 1e-5 * abs(ref), (n, d, r, got, ref)
    if n < 2:
        return
    _, S = oracle.mean_cov(X)
    if np.linalg.cond(S) > 1e8:
        return
    hs = np.array([0.5, 1.0, 2.0]) * scale
    np.testing.assert_allclose(ctx.lscv_h_scores(Xd, hs), oracle.lscv_h_scores(X, hs), rtol=1e-5)
    Hs = [datagen.vech(h * h * S) for h in hs]
    np.testing.assert_allclose(ctx.lscv_H_scores(Xd, Hs), [oracle.lscv_H_score(X, v) for v in Hs], rtol=1e-5)
    Y = _data(max(1, n // 3), d, n + 7)
    H = datagen.unvech(Hs[1], d)
    ref = oracle.kde_eval(X, Y, H)
    # densities: relative 1e-5, or 1e-7 of the peak for far-tail queries (fp32 exponent arguments
    # of a far query carry an absolute error proportional to its distance)
    np.testing.assert_allclose(ctx.evaluate(Xd, kb.to_device(Y), H), ref, rtol=1e-5, atol=max(1e-7 * ref.max(), 1e-300))
