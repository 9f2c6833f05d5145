"""Two ranks on one GPU through the library's SPMD path.

NCCL refuses two ranks on the same device, so the ranks use the library's host-staged test
transport (kde_set_host_allreduce: the int64 partial sums of each pass are summed with a gloo
all-reduce).  Everything else is the multi-GPU code path: each rank evaluates only its contiguous
tile range, the all-reduced exact fixed-point sums feed the host decisions (PLUGIN chain, grid
argmin, Nelder-Mead) on every rank, and every rank must return results bit-identical to the
single-GPU run."""
import json
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

import datagen  # noqa: E402
import paper_1505_01998_b200 as kb  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload(ctx):
    x = kb.to_device(datagen.sample_mixture("skewed", 20000, 61))
    X = kb.to_device(datagen.sample_mixture("C3", 3000, 62))
    h, tr = ctx.plugin_h(x)
    sel = ctx.select_bandwidth(kb.LSCV_H, X, max_iter=60)
    selh = ctx.select_bandwidth(kb.LSCV_h, X, n_grid=40)
    return {
        "plugin": [h, tr["psi6"], tr["psi4"]],
        "lscv_h": ctx.lscv_h_scores(X, np.linspace(0.05, 1.0, 20)).tolist(),
        "lscv_H": ctx.lscv_H_scores(X, [[0.05, 0.01, 0.04], [0.2, -0.02, 0.1]]).tolist(),
        "nm": [sel["vechH"].tolist(), sel["objective"], sel["iterations"]],
        "grid": [selh["h"], selh["iterations"]],
        "raw": [list(f.key()) for f in ctx.raw_sums(kb.SUM_PSI4, x, [0.3])],
    }


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = kb.Context.distributed_host(device=0)
    res = _workload(ctx)
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump(res, f)
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ranks_sharing_one_gpu_match_the_single_gpu_run(tmp_path, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    ranks = [json.load(open(tmp_path / f"r{r}.json")) for r in range(world)]
    ctx = kb.Context()
    single = json.loads(json.dumps(_workload(ctx)))
    ctx.close()
    for r in ranks:
        assert r == single
