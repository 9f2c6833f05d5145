"""Printed values of the paper / SPEC (tests/golden/paper_examples.json) against the oracle (CPU)
and, when a GPU is present, the library."""
import json
import math
import os

import numpy as np
import pytest

import oracle

EX = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "paper_examples.json")))


def test_vech_example():
    e = EX["vech"]
    assert list(oracle.vech(np.array(e["A"]))) == e["vech"]


def test_kernel_constants():
    e = EX["kernel_constants"]
    assert oracle.kernel_deriv(6, 0.0) == pytest.approx(e["K6_0"], rel=1e-15)
    assert oracle.kernel_deriv(4, 0.0) == pytest.approx(e["K4_0"], rel=1e-15)
    assert 1 / (2 * math.sqrt(math.pi)) == pytest.approx(e["R_K"], rel=1e-15)


def test_spec_lscv_values():
    e = EX["lscv_H_n2_equal_points"]
    assert oracle.lscv_H_score(np.array(e["X"]), e["vechH"]) == pytest.approx(e["g"], abs=1e-10)
    # T~(0) = (K*K)(0) - 2K(0) at Sigma = 1, h = 1: the g of n=2 equal points minus the R(K)/n term
    n = 2
    T0 = (e["g"] - 0.5 / (2 * math.sqrt(math.pi))) * n * n / 2
    assert T0 == pytest.approx(EX["lscv_h_T0"]["T0"], abs=1e-9)


def test_h0_and_H_start():
    assert oracle.lscv_h0(EX["h0_d1"]["n"], 1) == pytest.approx(EX["h0_d1"]["h0"], rel=1e-9)
    # H_start scales as n^{-1/5} Sigma^{1/2}: n=2 samples {-1, 1} have Sigma = 2
    Hs = oracle.H_start(np.array([[-1.0, 1.0]]))[0, 0]
    assert Hs == pytest.approx(EX["H_start_d1"]["H"] * 2 ** -0.2 * math.sqrt(2.0), rel=1e-9)


def test_toy_data_plugin_is_finite_and_equivariant():
    x = np.array(EX["toy_data"]["x"])
    t = oracle.plugin(x)
    assert t["psi6"] < 0 < t["psi4"] and t["h"] > 0
    assert oracle.plugin(2 * x)["h"] == pytest.approx(2 * t["h"], rel=1e-12)


@pytest.mark.gpu
def test_library_reproduces_printed_values():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1505_01998_b200 as kb
    ctx = kb.Context()
    e = EX["lscv_H_n2_equal_points"]
    g = ctx.lscv_H_scores(kb.to_device(np.array(e["X"])), [e["vechH"]])[0]
    assert g == pytest.approx(e["g"], abs=1e-8)
    x = np.array(EX["toy_data"]["x"])
    h, tr = ctx.plugin_h(kb.to_device(x))
    assert h == pytest.approx(oracle.plugin(x)["h"], rel=1e-5)
    # max_iter = 0: the best vertex of the initial simplex built on H_start (Eq. 35, reading Z8)
    X3 = np.array([[-1.0, 1.0, 0.3]])
    r = ctx.select_bandwidth(kb.LSCV_H, kb.to_device(X3), max_iter=0)
    ref = oracle.lscv_H_select(X3, max_iter=0)
    assert r["vechH"][0] == pytest.approx(ref["x"][0], rel=1e-12)
