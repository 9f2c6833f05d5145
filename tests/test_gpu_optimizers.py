"""GPU parity for the optimizer variants of SURVEY §8(f) f4: LSCV_h grid refinement and
multi-start Nelder-Mead for LSCV_H (lockstep runs sharing one GPU batch per round)."""
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


def test_lscv_h_refinement_matches_oracle(ctx):
    X = datagen.sample_mixture("bimodal", 2500, 31)
    got = ctx.select_bandwidth(kb.LSCV_h, kb.to_device(X), n_grid=64, refine_steps=6, refine_tol=1e-9)
    ref = oracle.lscv_h_select(X, n_grid=64, refine_steps=6, refine_tol=1e-9)
    assert got["iterations"] == ref["index"]
    g_or_at_gpu = oracle.lscv_h_scores(X, [got["h"]])[0]
    eps = abs(got["objective"] - g_or_at_gpu) / abs(g_or_at_gpu)
    assert eps < 1e-5
    # same h to 1e-4, or indistinguishable objective (tie rule)
    assert abs(got["h"] - ref["h"]) / ref["h"] < 1e-4 or g_or_at_gpu - ref["objective"] <= 2 * eps * abs(ref["objective"])
    assert got["objective"] <= ctx.lscv_h_scores(kb.to_device(X), [ref["grid"][ref["index"]]])[0]


def test_multistart_nm_matches_oracle(ctx):
    X = datagen.sample_mixture("C3", 500, 17)
    got = ctx.select_bandwidth(kb.LSCV_H, kb.to_device(X), max_iter=300, nm_starts=3)
    ref = oracle.lscv_H_select(X, max_iter=300, nm_starts=3)
    Hg = datagen.unvech(got["vechH"], 2)
    g_or = oracle.lscv_H_score(X, Hg)
    eps = abs(got["objective"] - g_or) / abs(g_or)
    assert eps < 1e-5
    close = np.max(np.abs(Hg - ref["H"])) / np.max(np.diag(ref["H"])) < 1e-4
    assert close or g_or <= ref["f"] + max(2 * eps, 1e-7) * abs(ref["f"])
    single = ctx.select_bandwidth(kb.LSCV_H, kb.to_device(X), max_iter=300, nm_starts=1)
    assert got["objective"] <= single["objective"]


def test_multistart_single_equals_default(ctx):
    X = kb.to_device(datagen.sample_mixture("C3", 1500, 5))
    a = ctx.select_bandwidth(kb.LSCV_H, X, max_iter=100)
    b = ctx.select_bandwidth(kb.LSCV_H, X, max_iter=100, nm_starts=1, speculative=1)
    assert np.array_equal(a["vechH"], b["vechH"]) and a["iterations"] == b["iterations"]


def test_multistart_nm_on_dirty_caller_workspace():
    # Regression: the prep flags must sit at an offset that does not depend on a batch's output
    # count (Nelder-Mead prepares the data once, then launches batches of 4..16 candidates).  A
    # caller workspace filled with 0xFF bytes exposes any read of a flag the prep did not write.
    X = datagen.sample_mixture("C3", 4000, 23)
    clean = kb.Context()
    ref = clean.select_bandwidth(kb.LSCV_H, X, max_iter=60, nm_starts=4)
    clean.close()
    c = kb.Context()
    ws = torch.full((kb.lib().kde_workspace_bytes(4000, 2, 64),), 255, dtype=torch.uint8, device="cuda")
    c.set_workspace(ws)
    got = c.select_bandwidth(kb.LSCV_H, X, max_iter=60, nm_starts=4)
    c.close()
    assert np.array_equal(got["vechH"], ref["vechH"]) and got["objective"] == ref["objective"]


@pytest.mark.parametrize("name,n,d,seed,max_iter", [("C3", 3000, 2, 41, 500), ("C3", 700, 2, 42, 40),
                                                     ("C5", 1200, 3, 43, 500), ("C5", 900, 4, 44, 200),
                                                     ("bimodal", 800, 1, 45, 500), ("C3", 50, 2, 46, 500),
                                                     ("C3", 5, 2, 47, 500)])
def test_device_nm_loop_equals_host_loop(ctx, name, n, d, seed, max_iter):
    # The device-resident Nelder-Mead (one CUDA graph, conditional WHILE node) runs the state
    # machine of kde_nm.cuh without FMA contraction, so on the same objective values it must take
    # exactly the host loop's decisions: identical H bits, objective, iterations, evaluations.
    X = datagen.sample_mixture(name, n, seed)[:d]
    Xd = kb.to_device(X)
    dev = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=max_iter, nm_loop=0)
    host = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=max_iter, nm_loop=1)
    assert np.array_equal(dev["vechH"], host["vechH"])
    assert dev["objective"] == host["objective"]
    for k in ("iterations", "evaluations", "stop_reason"):
        assert dev[k] == host[k], k
    # replayed graph on a second call (same key) gives the same result
    again = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=max_iter, nm_loop=0)
    assert np.array_equal(again["vechH"], dev["vechH"]) and again["evaluations"] == dev["evaluations"]


def test_device_nm_with_non_pd_proposals(ctx):
    # A huge penalty-side start (max_iter small, near-singular data) makes the simplex propose
    # non-PD matrices: those get the penalty on the device exactly as on the host.
    t = np.linspace(0.0, 1.0, 400)
    X = np.vstack([t, t + 1e-3 * np.sin(37.0 * t)])
    Xd = kb.to_device(X)
    dev = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=200, nm_loop=0)
    host = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=200, nm_loop=1)
    assert np.array_equal(dev["vechH"], host["vechH"]) and dev["evaluations"] == host["evaluations"]


@pytest.mark.parametrize("d,n,seed,max_iter", [(5, 400, 51, 60), (6, 300, 52, 40)])
def test_device_nm_large_d_equals_host_loop(ctx, d, n, seed, max_iter):
    # P = d(d+1)/2 > 10: the decision runs on the global state block (the one-thread decide kernel)
    X = np.random.default_rng(seed).normal(size=(d, n)) * np.linspace(0.5, 2.0, d)[:, None]
    Xd = kb.to_device(X)
    dev = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=max_iter, nm_loop=0)
    host = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=max_iter, nm_loop=1)
    assert np.array_equal(dev["vechH"], host["vechH"]) and dev["objective"] == host["objective"]
    for k in ("iterations", "evaluations", "stop_reason"):
        assert dev[k] == host[k], k


@pytest.mark.parametrize("env", [{"KDE_DEBUG_NM_UNROLL": "1"}, {"KDE_DEBUG_NM_UNROLL": "3"},
                                 {"KDE_DEBUG_NM_PDL": "0"}, {"KDE_DEBUG_NM_UNROLL": "16"}])
def test_device_nm_loop_shape_does_not_change_the_search(ctx, env):
    # Rounds per loop condition (the decisions after the stopping one are no-ops) and the programmatic
    # launches change only the schedule: the same search, bit for bit.
    import os
    Xd = kb.to_device(datagen.sample_mixture("C3", 2000, 61))
    ref = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=500, nm_loop=0)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        got = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=500, nm_loop=0)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
    assert np.array_equal(got["vechH"], ref["vechH"]) and got["objective"] == ref["objective"]
    for k in ("iterations", "evaluations", "stop_reason"):
        assert got[k] == ref[k], k


def test_device_nm_loop_equals_host_loop_seeded_sweep(ctx):
    # 24 seeded small problems (d = 1..4, n = 4..500, stretched / correlated / near-degenerate data):
    # the device-resident loop and the host loop take identical decisions on every one.
    rng = np.random.default_rng(2024)
    for case in range(24):
        d = int(rng.integers(1, 5))
        n = int(rng.integers(4, 500))
        A = rng.normal(size=(d, d)) * (1.0 + 3.0 * rng.random())
        X = A @ rng.standard_t(4, size=(d, n)) + rng.normal(size=(d, 1))
        if case % 6 == 5:            # near-degenerate covariance: non-PD proposals are likely
            X[-1] = X[0] + 1e-3 * rng.normal(size=n)
        Xd = kb.to_device(X)
        try:
            dev = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=150, nm_loop=0)
        except kb.KDEError as e:
            with pytest.raises(kb.KDEError) as e2:
                ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=150, nm_loop=1)
            assert e2.value.status == e.status
            continue
        host = ctx.select_bandwidth(kb.LSCV_H, Xd, max_iter=150, nm_loop=1)
        assert np.array_equal(dev["vechH"], host["vechH"]), (case, d, n)
        assert dev["objective"] == host["objective"] and dev["evaluations"] == host["evaluations"], (case, d, n)
