#!/bin/bash
# Evidence for the Psi path: GPU tests, full bench, ncu launch list, ncu --set full of Psi6 and Psi4.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_under_ncu.log 2>&1
for s in 2 3; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s $s -c 1 \
    -o gpurun_out/prof_psi_s$s -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_s$s.log 2>&1
done
