#!/bin/bash
# One GPU session: parity tests, psi diagnostics, bench.  Output under gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
for n in 131109 40000; do for T in 512 2048; do KDE_DEBUG_PSI_TILE=$T timeout 300 python tests/diag/dbg_psi2.py $n 0.2; done; done
timeout 600 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
