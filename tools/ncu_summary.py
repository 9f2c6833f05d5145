"""Summarise ncu output into profiles/ (committed evidence).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py full <report.ncu-rep> <out_prefix> [expected_evals_per_launch ...]
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__grid_size", "grid"), ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs, CTAs/SM)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe inst %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe inst %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe cycles %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe cycles %"),
    ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio_throttle / issue"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_pipe_throttle / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not_selected / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier / issue"),
]

BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
    tot = {}
    for r in rows[hdr + 1:]:
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        k = r[ki].split("(")[0]
        tot.setdefault(k, [0.0, 0])
        tot[k][0] += v
        tot[k][1] += 1
    S = sum(v[0] for v in tot.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list: `{path}`\n\n`ncu --metrics gpu__time_duration.sum --clock-control none` "
                "(cold-cache, serialised launches: compare shares, not absolutes)\n\n")
        f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1][0]):
            f.write(f"| `{k}` | {v[1]} | {v[0]:.3f} | {100 * v[0] / S:.2f}% |\n")
    print(open(out).read())


def full(rep, prefix, expected):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for key, label in KEYS:
            if key in h:
                i = h.index(key)
                d[key] = {"value": r[i], "unit": units[i], "label": label}
        kernels.append(d)
    md = [f"# ncu --set full summary: `{rep}`\n"]
    out = []
    for n, d in enumerate(kernels):
        md.append(f"\n## {d['kernel'][:120]}\n\n| metric | value |\n|---|---|")
        for key, label in KEYS:
            if key in d:
                md.append(f"| {label} (`{key}`) | {d[key]['value']} {d[key]['unit']} |")
        rb = d.get("dram__bytes_read.sum")
        wb = d.get("dram__bytes_write.sum")
        traffic = None
        try:
            traffic = float(rb["value"].replace(",", "")) * BYTES.get(rb["unit"], 1) + \
                float(wb["value"].replace(",", "")) * BYTES.get(wb["unit"], 1)
        except Exception:
            pass
        md.append(f"| DRAM read+write per launch | {traffic} bytes |")
        if n < len(expected):
            try:
                dur = float(d["gpu__time_duration.sum"]["value"].replace(",", ""))
                unit = d["gpu__time_duration.sum"]["unit"]
                sec = dur * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1, "s": 1}[unit]
                md.append(f"| algorithmic evals / duration | {float(expected[n]) / sec:.4e} evals/s |")
            except Exception:
                pass
        out.append({"kernel": d["kernel"], "dram_bytes_per_launch": traffic,
                    **{k: d[k]["value"] + " " + d[k]["unit"] for k, _ in KEYS if k in d}})
    open(prefix + ".md", "w").write("\n".join(md) + "\n")
    json.dump(out, open(prefix + ".json", "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4:])
