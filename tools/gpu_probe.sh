#!/bin/bash
# e2e breakdown + parity + bench + Psi ncu (both passes).  Output under gpurun_out/.
mkdir -p gpurun_out
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_under_ncu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 2 -c 2 \
    -o gpurun_out/prof_psi -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_psi.log 2>&1
tail -2 gpurun_out/pytest_gpu.txt; cat gpurun_out/e2e_probe.jsonl gpurun_out/bench.json; tail -3 gpurun_out/ncu_psi.log
