#!/usr/bin/env python
"""Benchmark of the all-pairs kernel-sum engine (arxiv 1505.01998) on B200.

Workload (BASELINE.json metric "pair-kernel evals/s and time-to-bandwidth at n=2^20"):
config C4 = PLUGIN bandwidth of n = 2^20 samples from the Marron–Wand #2 skewed mixture
(datagen, seed 4).  One step = one full kde_plugin_h call: moments, data prep, the Psi_6(g1)
and Psi_4(g2) all-pairs passes (2 x 549,755,289,600 pair-kernel evaluations), the NCCL
all-reduce (N > 1) and the host scalar chain.  value = algorithmic evals / device time, summed
over steps, max over ranks.  L2 is flushed (256 MiB write) between timed steps, outside the
timed events.  `e2e` repeats the step through the public API from pinned host memory.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

`--gpus N` with N > 1 outside torchrun re-executes itself under `torch.distributed.run`
(127.0.0.1, a free port), so both launch forms run N ranks; under torchrun the world size must
equal --gpus.  `--dry-run` runs the same multi-rank plumbing on CPU (gloo, no kernels): every rank
reports its tile range of the pair partition, rank 0 prints one JSON line (tests/test_bench_cli.py).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_C4 = 1 << 20
METRIC = "pair-kernel evals/s (PLUGIN n=2^20, Psi6+Psi4 passes)"
MUFU_PER_CLK_SM = 16          # MUFU.EX2 lanes per clock per SM (measured 15.98, tools/peaks.cu)
SM_MAX_MHZ = 1965.0


def evals_per_step(n: int) -> float:
    return 2.0 * n * (n - 1) / 2.0


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, gpu: int):
        self.gpu, self.samples, self.proc, self.thread = gpu, [], None, None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[3 + k].lower().startswith("active")})
        loaded = [v for v in sm if v > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.samples)}


def cpu_baseline_sample(x: np.ndarray, g: tuple, seconds: float = 12.0):
    """Time the fp64 oracle (as it stands) on a bounded row sample of the same workload."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    n = x.size
    rows = 64
    pairs = 0
    t0 = time.perf_counter()
    i0 = 0
    # grow the sample until ~seconds of CPU time per pass
    while time.perf_counter() - t0 < seconds and i0 < n:
        hi = min(n, i0 + rows * cores)
        chunks = [(i0 + k * rows, min(hi, i0 + (k + 1) * rows)) for k in range(cores)]
        chunks = [c for c in chunks if c[0] < c[1]]
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=cores) as ex:
            list(ex.map(lambda c: (oracle.psi_pairsum(x, 6, g[0], rows=c), oracle.psi_pairsum(x, 4, g[1], rows=c)), chunks))
        pairs += 2 * sum((n - 1 - i) for a, b in chunks for i in range(a, b))
        i0 = hi
    dt = time.perf_counter() - t0
    return {"value": pairs / dt, "unit": "evals/s", "cores": cores, "kind": "oracle", "evals": pairs,
            "sample": f"rows 0..{i0} of C4 (all j>i), Psi6(g1)+Psi4(g2) pair sums, {pairs:.3e} evals in {dt:.1f}s"}


def load_traffic():
    p = os.path.join(ROOT, "profiles", "ncu_psi_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def run_reference(args, rank, world):
    """The reference arm (tier rules): the fp64 oracle as it stands, timed on this box's host
    cores; each step is a bounded row sample of the C4 workload whose wall time is MEASURED
    (ms_per_step is that measured time, not an extrapolation to the full step)."""
    if rank != 0:
        return
    import datagen
    x = datagen.config_data("C4")[0]
    # g1, g2 of this sample's PLUGIN chain, as the oracle computed them once at full size
    # (tests/golden/make_golden.py, which calls only oracle/); each step times the oracle's two
    # pair sums on a bounded row sample at those bandwidths.
    tr = json.load(open(os.path.join(ROOT, "tests", "golden", "C4_plugin.json")))["trace"]
    g1, g2 = tr["g1"], tr["g2"]
    times, vals, evals = [], [], []
    per_step_s = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = cpu_baseline_sample(x, (g1, g2), seconds=per_step_s)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            vals.append(r["value"])
            times.append(dt * 1e3)
            evals.append(r["evals"])
    v = sum(evals) / (sum(times) / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.median(times),
            "ms_per_step_basis": "measured wall time of one bounded-sample step (oracle on host cores)",
            "full_step_ms_extrapolated": evals_per_step(x.size) / v * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "C4 PLUGIN n=2^20 skewed mixture (MW#2)", "n": x.size,
                                            "sample_evals_per_step": statistics.median(evals)},
            "cpu_baseline": {"value": v, "unit": "evals/s", "cores": r["cores"], "kind": "oracle", "sample": r["sample"]},
            "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(n: int):
    """`python bench.py --gpus N` (N > 1) outside torchrun: become `torch.distributed.run` with N
    ranks on this node (the driver's own launch form), so N really is the world size."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def run_dry(args, rank, world):
    """CPU check of the N-rank plumbing (gloo): rendezvous, each rank's contiguous tile range of
    the C4 pair partition (the library's own kde_shard_tiles: round-robin chunks), barrier and max-over-ranks
    reduction as in the timed path; rank 0 prints the JSON line.  No kernels run."""
    import torch
    import torch.distributed as dist
    import paper_1505_01998_b200 as kb
    if world > 1:
        dist.init_process_group("gloo")
    T, total, cnt, chunk = kb.shard_tiles(kb.SUM_PSI6, args.n, 1, rank, world)
    t = torch.tensor([float(cnt), float(rank)], dtype=torch.float64)
    mine = (cnt, chunk, kb.shard_tile(0, rank, world) if cnt else None)
    ranges = [None] * world
    if world > 1:
        dist.barrier()
        dist.all_gather_object(ranges, mine)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    else:
        ranges = [mine]
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "evals/s", "n_gpus": world, "steps": 0,
                          "warmup": 0, "dry_run": True, "scaling": "strong",
                          "config": {"workload": "C4 PLUGIN n=2^20 skewed mixture (MW#2), seed 4", "n": args.n,
                                     "parallelism": f"pair-range x{world}", "tile": T, "tiles": total,
                                     "rank_tiles_chunk_first": ranges, "max_rank_tiles": float(t[0])}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_C4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="CPU check of the N-rank plumbing (gloo, no kernels)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        run_dry(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    import datagen
    import paper_1505_01998_b200 as kb

    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        ctx = kb.Context.distributed(device=local, profiling=True)
    else:
        ctx = kb.Context(device=local, profiling=True)

    x_host = datagen.config_data("C4", n=args.n)            # identical on every rank
    n = x_host.shape[1]
    x_dev = kb.to_device(x_host)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        h, tr = ctx.plugin_h(x_dev)

    # ------------------------------------------------------------ device-resident timing
    sampler = ClockSampler(local)
    sampler.start()
    barrier()
    step_ms, pair_ms, pair_launches, kernel_launches, pair_evals = [], 0.0, 0, 0, 0.0
    for _ in range(args.steps):
        flush.random_(0, 255)                                 # L2 flush, outside the events
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h, tr = ctx.plugin_h(x_dev)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        prof = ctx.last_profile()
        pair_ms += prof["pair_ms"]
        pair_launches += prof["pair_launches"]
        kernel_launches += prof["kernel_launches"]
        pair_evals += prof["pair_evals"]        # MUFU-evaluated pairs (skipped far tiles excluded)
    kappa = ctx.last_psi_kappa()
    barrier()
    clocks = sampler.stop()
    clocks_per_rank = [clocks]
    if world > 1:
        clocks_per_rank = [None] * world
        dist.all_gather_object(clocks_per_rank, {k: clocks.get(k) for k in ("sm_mhz", "sm_max_mhz", "reasons")})
    total_ms = sum(step_ms)
    # per-rank MUFU throughput of the pair kernels (evaluated pairs / their device time); the
    # roofline reports the slowest rank
    ach_rank = pair_evals / (pair_ms / 1e3) if pair_ms > 0 else 0.0
    t = torch.tensor([total_ms, pair_ms, -ach_rank], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, pair_ms_max, achieved = float(t[0]), float(t[1]), -float(t[2])
    evals = evals_per_step(n) * args.steps
    value = evals / (total_ms / 1e3)

    # ------------------------------------------------------------ end-to-end (host buffers)
    # The C-ABI call itself takes the pinned HOST buffer: the library copies it to the GPU on
    # its stream inside the call and returns h (and the trace) in host memory.
    e2e = None
    if not args.no_e2e:
        x_pin = torch.from_numpy(x_host).pin_memory()
        barrier()
        ee = []
        for _ in range(max(1, min(args.steps, 10))):
            flush.random_(0, 255)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            hh, _ = ctx.plugin_h(x_pin)                    # H2D, the whole path, D2H of h
            ee.append(time.perf_counter() - t0)
        tt = torch.tensor([sum(ee)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": evals_per_step(n) * len(ee) / float(tt[0]), "unit": "evals/s",
               "h2d_bytes_per_step": int(x_host.nbytes), "d2h_bytes_per_step": 8 * 8}

    if rank == 0:
        per_launch_ms = pair_ms_max / max(1, pair_launches)
        evaluated_fraction = pair_evals * world / (evals_per_step(n) / 2 * pair_launches) if pair_launches else None
        peak = MUFU_PER_CLK_SM * torch.cuda.get_device_properties(local).multi_processor_count * SM_MAX_MHZ * 1e6
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "C4 PLUGIN n=2^20 skewed mixture (MW#2), seed 4", "n": n,
                       "parallelism": f"pair-range x{world}", "l2": "flushed (256 MiB write) between steps",
                       "h": h, "time_to_bandwidth_ms": total_ms / args.steps,
                       "psi_kappa": kappa, "psi_fp64_passes": ctx.last_fp64_passes(),
                       "evaluated_pair_fraction": evaluated_fraction},
            "roofline": {"bound": "alu", "pipe": "MUFU.EX2 (1 per evaluated pair; far tiles whose terms are exactly 0 or provably < 1e-9 of Psi-hat are skipped and not counted, DESIGN.md 3.11)",
                         "achieved": achieved / 1e12,
                         "peak": peak / 1e12, "unit": "Tex2/s", "frac": achieved / peak,
                         "traffic": load_traffic(), "kernel": "pair_kernel<FPsi<6|4,8>>",
                         "peak_basis": "16 MUFU.EX2/clk/SM x SMs x 1965 MHz (guide unit counts; tools/peaks.cu measured 4.646e12/s)"},
            "clocks": clocks,
            "gpu_launches": kernel_launches,
            "pair_ms_per_launch": per_launch_ms,
            "e2e": e2e,
        }
        if world > 1:
            line["clocks_per_rank"] = clocks_per_rank
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline_sample(x_host[0], (tr["g1"], tr["g2"]))
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
