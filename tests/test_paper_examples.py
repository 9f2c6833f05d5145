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


def test_plugin_x123_worked_trace():
    # Every step of the PLUGIN chain (Eq. 11-18) against the independently computed mpmath trace:
    # a wrong root (1/9, 1/7, 1/5), a dropped -2 or mu2 factor, or a wrong K^(r)(0) fails here.
    e = EX["plugin_x123_trace"]
    t = oracle.plugin(np.array(e["x"]))
    for k in ("V_hat", "sigma_hat", "psi8_ns", "g1", "psi6", "g2", "psi4", "h"):
        assert t[k] == pytest.approx(e[k], rel=1e-12), k


def test_lscv_h0_hand_values_d_gt_1():
    # Eq. 25 as written, reading Z3: h0 = (4/(d^3 (d+2) n))^{1/(d+4)} by hand.
    for c in EX["lscv_h0_hand"]["cases"]:
        d, n = c["d"], c["n"]
        ref = c["h0"] if "h0" in c else (c["num"] / (c["den"] * n)) ** (1.0 / (d + 4))
        assert oracle.lscv_h0(n, d) == pytest.approx(ref, rel=1e-13), (d, n)
    # the grid is bracketed by it (Eq. 27)
    hs = oracle.lscv_h_grid(32768, 2, 5)
    assert list(hs) == pytest.approx([0.125 / 4, 0.125 / 4 + 0.125 * 3.75 / 4 * 1, 0.125 / 4 + 0.125 * 3.75 / 4 * 2,
                                      0.125 / 4 + 0.125 * 3.75 / 4 * 3, 0.5], rel=1e-14)


@pytest.mark.parametrize("case", ["d2", "d3"])
def test_initial_simplex_hand_vertices(case):
    # Reading Z8: an off-diagonal entry that is 0 still gets a nonzero step 0.1*sqrt(H_aa H_bb).
    e = EX["nm_initial_simplex_hand"][case]
    d = 2 if case == "d2" else 3
    sim = oracle.initial_simplex(np.array(e["x0"]), d)
    assert len(sim) == len(e["vertices"])
    for v, ref in zip(sim, e["vertices"]):
        np.testing.assert_allclose(v, ref, rtol=1e-15, atol=1e-15)


def test_nm_starts_scale_the_initial_simplex_by_powers_of_4():
    # Row f4 multi-start: run k starts from the initial simplex scaled by 4^-k; the best run
    # (ties -> earlier) is returned.  Checked on the evaluation trace: run 2's first m+1
    # evaluations are the hand-scaled vertices x_k / 4.
    X = np.array([[0.0, 0.4, 1.1, 1.5, 2.6, 3.0, 3.2, 4.4], [0.3, -0.2, 0.9, 0.1, 1.7, 1.2, 2.5, 2.1]])
    t1, t2 = [], []
    r1 = oracle.lscv_H_select(X, max_iter=30, trace=t1)
    r2 = oracle.lscv_H_select(X, max_iter=30, trace=t2, nm_starts=2)
    L = len(t1)
    for a, b in zip(t1, t2[:L]):
        np.testing.assert_array_equal(a[0], b[0])
    sim0 = oracle.initial_simplex(oracle.vech(r1["H_start"]), 2)
    for k, v in enumerate(sim0):
        np.testing.assert_allclose(t2[L + k][0], v / 4.0, rtol=1e-15)
    run2 = [f for _, f in t2[L:]]
    assert r2["f"] == min(r1["f"], r2["f"]) and r2["f"] <= r1["f"]
    assert r2["f"] in run2 or r2["f"] == r1["f"]


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
