#!/bin/bash
# GPU eval tests + F2 with the bounded far-tile skip (default) and without (KDE_DEBUG_EVAL_NOSKIP=1).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eval.py tests/test_gpu_golden.py -k "eval or f2" -m gpu -q > gpurun_out/pytest_eval.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_eval.txt
timeout 600 python tools/bench_configs.py F2 > gpurun_out/f2_skip.jsonl 2>&1
KDE_DEBUG_EVAL_NOSKIP=1 timeout 600 python tools/bench_configs.py F2 > gpurun_out/f2_noskip.jsonl 2>&1
tail -3 gpurun_out/pytest_eval.txt; cut -c1-160 gpurun_out/f2_skip.jsonl gpurun_out/f2_noskip.jsonl
