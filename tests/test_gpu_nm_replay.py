"""Nelder–Mead decision-path parity (SURVEY §8(c) c5 "replay parity").

The library's NM (C++, kde_host.cpp) and the oracle's NM (Python, oracle.nelder_mead, itself
pinned step for step to scipy in tests/test_oracle_lscv.py) are independent implementations of
the reading-Z8 spec.  Three checks on seeded inputs:
  (a) the oracle NM driven by the GPU objective takes exactly the library's path (same
      iterations, same final vech to rounding of the start point): pins the library's host logic;
  (b) replay: every H that path visits has GPU objective within 1e-5 of the fp64 oracle's;
  (c) the all-oracle NM (fp64 objective) takes the same decision sequence: the fp32-term
      objective changes no decision on these inputs.
"""
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


@pytest.mark.parametrize("mix,d,n,seed,max_iter", [("C3", 2, 1500, 41, 300), ("C5", 3, 700, 42, 150)])
def test_nm_path_library_gpu_driven_and_oracle_agree(mix, d, n, seed, max_iter):
    X = datagen.sample_mixture(mix, n, seed)[:d]
    ctx = kb.Context()
    Xd = kb.to_device(X)
    lib_sel = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=max_iter)

    sim0 = oracle.initial_simplex(oracle.vech(oracle.H_start(X)), d)
    f_gpu = lambda v: float(ctx.lscv_H_scores(Xd, [v])[0])
    tg = []
    gpu_driven = oracle.nelder_mead(f_gpu, sim0, max_iter=max_iter, trace=tg)
    ctx.close()
    # (a) same path as the library's own NM
    assert lib_sel["iterations"] == gpu_driven["iterations"]
    assert np.max(np.abs(lib_sel["vechH"] - gpu_driven["x"])) <= 1e-10 * np.max(np.abs(gpu_driven["x"]))
    # (the start points differ in the last bits: Jacobi vs Denman-Beavers square roots)
    assert abs(lib_sel["objective"] - gpu_driven["f"]) <= 1e-9 * abs(gpu_driven["f"])
    # (b) replay parity of every visited candidate
    f_or = [oracle.lscv_H_score(X, x, threads=THREADS) for x, _ in tg]
    for (x, fg), fo in zip(tg, f_or):
        if fo == oracle.PENALTY:
            assert fg == fo
        else:
            assert abs(fg - fo) <= 1e-5 * abs(fo), (x, fg, fo)
    # (c) the fp64 oracle NM makes the same decisions (identical visited points)
    to = []
    oracle.nelder_mead(lambda v: oracle.lscv_H_score(X, v, threads=THREADS), sim0, max_iter=max_iter, trace=to)
    assert len(to) == len(tg)
    for (xo, _), (xg, _) in zip(to, tg):
        assert np.array_equal(xo, xg)


@pytest.mark.parametrize("mix,d,n,seed,max_iter", [("C3", 2, 1200, 43, 300), ("C5", 3, 600, 44, 200)])
def test_nm_fp64_term_mode_reproduces_the_oracle_search(mix, d, n, seed, max_iter):
    # SURVEY c5's optional exact-parity mode: with kde_set_precision(1) every g(H) of the search runs
    # with fp64 terms (host loop), so the library's search and the all-oracle search make the same
    # decisions and end at the same H (to the last bits of the start point's square root).
    X = datagen.sample_mixture(mix, n, seed)[:d]
    ctx = kb.Context()
    ctx.set_precision(1)
    got = ctx.select_bandwidth(kb.LSCV_H, kb.to_device(X), max_iter=max_iter)
    ctx.close()
    sim0 = oracle.initial_simplex(oracle.vech(oracle.H_start(X)), d)
    ref = oracle.nelder_mead(lambda v: oracle.lscv_H_score(X, v, threads=THREADS), sim0, max_iter=max_iter)
    assert got["iterations"] == ref["iterations"]
    assert np.max(np.abs(got["vechH"] - ref["x"])) <= 1e-9 * np.max(np.abs(ref["x"]))
    assert abs(got["objective"] - ref["f"]) <= 1e-10 * abs(ref["f"])


@pytest.mark.parametrize("mix,d,n,seed,max_iter", [("C3", 2, 900, 45, 300), ("C5", 3, 500, 46, 200)])
def test_nm_cholesky_parametrisation_matches_oracle(mix, d, n, seed, max_iter):
    # Row f4 variant (kde_select_opts.nm_param = 1: search over vech(L), H = L L^T).  With fp64 terms the
    # library's search equals the oracle's (same iterations, H to 1e-9); with the default fp32 terms the
    # selected H's fp64 objective is within the NM tolerance band of the oracle's optimum.
    X = datagen.sample_mixture(mix, n, seed)[:d]
    ref = oracle.lscv_H_select(X, max_iter=max_iter, param="chol", threads=THREADS)
    ctx = kb.Context()
    ctx.set_precision(1)
    exact = ctx.select_bandwidth(kb.LSCV_H, kb.to_device(X), max_iter=max_iter, nm_param=1)
    ctx.set_precision(0)
    fast = ctx.select_bandwidth(kb.LSCV_H, kb.to_device(X), max_iter=max_iter, nm_param=1)
    ctx.close()
    assert exact["iterations"] == ref["iterations"]
    Href = oracle.vech(ref["H"])
    assert np.max(np.abs(exact["vechH"] - Href)) <= 1e-9 * np.max(np.abs(Href))
    g_fast = oracle.lscv_H_score(X, fast["vechH"], threads=THREADS)
    assert g_fast <= ref["f"] + max(1e-7, 2e-6) * abs(ref["f"])
