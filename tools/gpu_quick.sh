#!/bin/bash
# Quick iteration: GPU tests, bench (no CPU baseline), ncu of the two Psi launches.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
grep -o '"ms_per_step": [0-9.]*\|"frac": [0-9.]*\|"e2e": {"value": [0-9.]*' gpurun_out/bench.json
if [ -z "$NO_NCU" ]; then
for s in 2 3; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s $s -c 1 \
    -o gpurun_out/prof_psi_s$s -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_s$s.log 2>&1
done
fi
