#!/bin/bash
# One GPU round trip with timestamps: GPU tests, smoke, bench, per-config report (args: configs).
mkdir -p gpurun_out
t0=$(date +%s)
stamp() { echo "[$(( $(date +%s) - t0 ))s] $*" >> gpurun_out/timeline.txt; }
: > gpurun_out/timeline.txt
stamp start
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
stamp pytest
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
stamp smoke
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
stamp bench
if [ -n "$CONFIGS" ]; then timeout 900 python tools/bench_configs.py $CONFIGS > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; stamp configs; fi
tail -8 gpurun_out/pytest_gpu.txt; cat gpurun_out/smoke.txt gpurun_out/bench.json gpurun_out/timeline.txt; tail -3 gpurun_out/bench.err
