"""The NCCL collective path of the library on one GPU: a single-rank communicator created from
an ncclUniqueId (dlopen of libnccl.so.2, ncclCommInitRank, ncclAllReduce of the int64 limbs on
the context stream) must leave every result bit-identical to the communicator-free path."""
import numpy as np
import pytest

import datagen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1505_01998_b200 as kb  # noqa: E402


def test_single_rank_nccl_path_is_bit_identical():
    plain = kb.Context()
    coll = kb.Context(rank=0, world=1, nccl_id=kb.nccl_unique_id())
    x = kb.to_device(datagen.sample_mixture("skewed", 20000, 3))
    X2 = kb.to_device(datagen.sample_mixture("C3", 4000, 3))
    assert plain.plugin_h(x) == coll.plugin_h(x)
    hs = np.linspace(0.05, 1.0, 40)
    np.testing.assert_array_equal(plain.lscv_h_scores(X2, hs), coll.lscv_h_scores(X2, hs))
    c = [[0.05, 0.01, 0.04], [0.2, -0.02, 0.1]]
    np.testing.assert_array_equal(plain.lscv_H_scores(X2, c), coll.lscv_H_scores(X2, c))
    np.testing.assert_array_equal(plain.lscv_h_scores_materialized(X2, hs, 4), coll.lscv_h_scores_materialized(X2, hs, 4))
    a = plain.select_bandwidth(kb.LSCV_H, X2, max_iter=60)
    b = coll.select_bandwidth(kb.LSCV_H, X2, max_iter=60)
    assert np.array_equal(a["vechH"], b["vechH"])
    coll.close()
    plain.close()


def test_distributed_context_world_one():
    import os
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        ctx = kb.Context.distributed(device=0)
        x = kb.to_device(datagen.config_data("C1"))
        h, _ = ctx.plugin_h(x)
        assert h == kb.Context().plugin_h(x)[0]
        ctx.close()
    finally:
        dist.destroy_process_group()
