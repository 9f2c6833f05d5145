mkdir -p gpurun_out
./tools/dp_overlap > gpurun_out/dp_overlap.txt 2>&1
KDE_DEBUG_NM_TRACE=1 python tools/c3_loop.py --reps 3 > gpurun_out/nm_trace.txt 2>&1
for u in 1 2 4 8; do echo "unroll $u: $(KDE_DEBUG_NM_UNROLL=$u python tools/c3_loop.py --reps 3 | tail -1)" >> gpurun_out/nm_trace.txt; done
echo "pdl off: $(KDE_DEBUG_NM_PDL=0 python tools/c3_loop.py --reps 3 | tail -1)" >> gpurun_out/nm_trace.txt
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:FLscvScalar -s 250 -c 1 -o gpurun_out/prof_c2_late -f python tools/bench_configs.py C2 --reps 1 > gpurun_out/ncu_c2_late.log 2>&1
timeout 1500 python tests/diag/psi_kappa.py > gpurun_out/psi_kappa.jsonl 2> gpurun_out/psi_kappa.err
timeout 1800 python tests/diag/fuzz_wide.py 600 7 6 4000 > gpurun_out/fuzz_wide.txt 2>&1
timeout 900 python tests/diag/fuzz_wide.py 150 11 16 2000 >> gpurun_out/fuzz_wide.txt 2>&1
ls -la gpurun_out | tail -12
