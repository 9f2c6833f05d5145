#!/bin/bash
# ncu evidence for every pair-kernel family (run under gpurun; 1 GPU).  Output in gpurun_out/;
# summarise with tools/ncu_summary.py into profiles/.
# usage: tools/gpu_prof.sh [psi] [lscv] [eval]
mkdir -p gpurun_out
if [[ " $* " == *" psi "* || $# -eq 0 ]]; then
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_under_ncu.log 2>&1
for s in 2 3; do   # the Psi6 and Psi4 launches of the first timed step
ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s $s -c 1 \
    -o gpurun_out/prof_psi_s$s -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_psi_s$s.log 2>&1
done
fi
if [[ " $* " == *" lscv "* || $# -eq 0 ]]; then
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:FLscvScalar -s 250 -c 1 \
    -o gpurun_out/prof_c2 -f python tools/bench_configs.py C2 --reps 1 > gpurun_out/ncu_c2.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:FLscvScalar -s 0 -c 1 \
    -o gpurun_out/prof_c5p -f python tools/bench_configs.py C5P --reps 1 > gpurun_out/ncu_c5p.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:FLscvScalar -s 30 -c 1 \
    -o gpurun_out/prof_c3 -f python tools/bench_configs.py C3 --reps 1 > gpurun_out/ncu_c3.log 2>&1
fi
if [[ " $* " == *" eval "* || $# -eq 0 ]]; then
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:eval_kernel -s 1 -c 1 \
    -o gpurun_out/prof_f2 -f python tools/bench_configs.py F2 --reps 2 > gpurun_out/ncu_f2.log 2>&1
fi
ls -la gpurun_out/*.ncu-rep
