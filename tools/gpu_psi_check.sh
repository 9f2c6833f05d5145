#!/bin/bash
# GPU check of the Psi path: parity/golden tests, kappa sweep, a short bench.
mkdir -p gpurun_out
timeout 600 python tests/diag/psi_kappa_sweep.py > gpurun_out/psi_kappa_sweep.jsonl 2> gpurun_out/psi_kappa_sweep.err
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
tail -15 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench2.json; tail -3 gpurun_out/psi_kappa_sweep.err
