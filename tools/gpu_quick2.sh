#!/bin/bash
# GPU tests + selected configs (CONFIGS) + bench, one gpurun call.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python tools/bench_configs.py ${CONFIGS:-C3 C2} > gpurun_out/configs_q.jsonl 2> gpurun_out/configs_q.err
[ -n "$BENCH" ] && timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.txt; cut -c1-200 gpurun_out/configs_q.jsonl
