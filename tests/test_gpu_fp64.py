"""fp64-term Psi mode (kde_set_precision): parity with the fp64 oracle where the
fp32-term path is limited (bandwidths far below the PLUGIN pilots), exactness of the shards, and
the PLUGIN chain in this mode."""
import math
import os

import numpy as np
import pytest

import datagen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1505_01998_b200 as kb  # noqa: E402

THREADS = len(os.sched_getaffinity(0))


@pytest.fixture(scope="module")
def ctx64():
    c = kb.Context()
    c.set_precision(True)
    yield c
    c.close()


def test_small_bandwidth_parity(ctx64):
    # n = 40 000, g = 0.02: the fp32-term path is off by 2.4e-5 here (profiles/r01_psi_accuracy.md)
    x = datagen.sample_mixture("skewed", 300000, 7)[:, :40000]
    ref = oracle.psi_pairsum(x[0], 6, 0.02, threads=THREADS)
    got = kb.fixed_value(ctx64.raw_sums(kb.SUM_PSI6, kb.to_device(x), [0.02])[0]) / math.sqrt(2 * math.pi)
    assert abs(got - ref) / abs(ref) < 1e-9


@pytest.mark.parametrize("n", [2, 3, 257, 1000, 3001])
def test_psi_r_fp64_matches_oracle(ctx64, n):
    x = datagen.sample_mixture("skewed", n, 70 + n)
    for r in (4, 6, 8):
        got = ctx64.psi_r(kb.to_device(x), r, [0.05, 0.4])
        for g, v in zip([0.05, 0.4], got):
            ref = oracle.psi_r(x[0], r, g)
            assert abs(v - ref) / abs(ref) < 1e-10, (n, r, g, v, ref)


def test_plugin_fp64_matches_oracle(ctx64):
    x = datagen.config_data("C1")
    h, tr = ctx64.plugin_h(kb.to_device(x))
    ref = oracle.plugin(x[0])
    for k in ("psi6", "psi4", "g2", "h"):
        assert abs(tr[k] - ref[k]) / abs(ref[k]) < 1e-10, k
    assert ctx64.plugin_h(kb.to_device(x)) == (h, tr)   # graph replay in this mode


def test_fp64_shards_add_up_exactly(ctx64):
    x = kb.to_device(datagen.sample_mixture("skewed", 5000, 71))
    full = ctx64.raw_sums(kb.SUM_PSI4, x, [0.1])
    acc = None
    for r in range(3):
        part = ctx64.raw_sums(kb.SUM_PSI4, x, [0.1], shard=(r, 3))
        acc = part if acc is None else [kb.fixed_add(a, b) for a, b in zip(acc, part)]
    assert [f.key() for f in acc] == [f.key() for f in full]
