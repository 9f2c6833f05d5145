"""bench.py's multi-rank launch (CPU): `python bench.py --gpus 2 --dry-run` re-executes itself under
torch.distributed.run with 2 ranks (gloo, no kernels) and reports n_gpus = 2 with the two ranks'
contiguous tile ranges covering the C4 pair partition."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_bench_gpus_2_runs_two_ranks():
    r = _run("--gpus", "2", "--dry-run")
    assert r["n_gpus"] == 2 and r["dry_run"]
    cfg = r["config"]
    (c0, k0, f0), (c1, k1, f1) = cfg["rank_tiles_chunk_first"]
    assert c0 + c1 == cfg["tiles"] and abs(c0 - c1) <= k0          # complete, balanced to one chunk
    assert k0 == k1 == 16 and f0 == 0 and f1 == 16                  # round-robin chunks of 16 tile ids
    assert cfg["max_rank_tiles"] == max(c0, c1)
    assert cfg["parallelism"] == "pair-range x2"


def test_bench_single_rank_dry_run():
    r = _run("--dry-run")
    cnt, _, first = r["config"]["rank_tiles_chunk_first"][0]
    assert r["n_gpus"] == 1 and cnt == r["config"]["tiles"] and first == 0
