#!/bin/bash
# One GPU round trip for the judged evidence: GPU tests, smoke, bench (+ reference arm), every config,
# launch list and ncu --set full of the pair kernels (C4 Psi6/Psi4, C2, C3, C5P).  Output in gpurun_out/.
mkdir -p gpurun_out
t0=$(date +%s)
stamp() { echo "[$(( $(date +%s) - t0 ))s] $*" >> gpurun_out/timeline.txt; }
: > gpurun_out/timeline.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
stamp pytest
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
stamp smoke
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
stamp bench
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
stamp bench_ref
timeout 1200 python tools/bench_configs.py ${CONFIGS:-C1 C4 C2 C5 C3 F1 F2 F3 F4} > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
stamp configs
if [ -z "$NO_NCU" ]; then bash tools/gpu_prof.sh psi lscv; stamp ncu; fi
tail -3 gpurun_out/pytest_gpu.txt; cat gpurun_out/smoke.txt; cut -c1-400 gpurun_out/bench.json; cat gpurun_out/timeline.txt
# summarise the ncu reports on the box (the .ncu-rep files would exceed gpurun's 64 MiB copy-back)
if [ -z "$NO_NCU" ]; then
  python tools/ncu_summary.py launches gpurun_out/launches.csv gpurun_out/launches.md > /dev/null 2>&1
  for r in gpurun_out/prof_*.ncu-rep; do python tools/ncu_summary.py full "$r" "${r%.ncu-rep}" > /dev/null 2>&1; done
  mkdir -p gpurun_out/reps && mv gpurun_out/prof_*.ncu-rep gpurun_out/reps/ 2>/dev/null
  [ -n "$KEEP_REPS" ] || rm -rf gpurun_out/reps
fi
du -sh gpurun_out
