#!/bin/bash
# Final evidence of the round (one gpurun call): tests, smoke, bench + reference arm, every config, launch
# list and ncu summaries (tools/gpu_evidence.sh), then the wide fuzz and the bounded-skip fuzz.
bash tools/gpu_evidence.sh
timeout 1200 python tests/diag/fuzz_wide.py 600 7 6 4000 > gpurun_out/fuzz_wide.txt 2>&1
timeout 600 python tests/diag/fuzz_wide.py 150 11 16 2000 >> gpurun_out/fuzz_wide.txt 2>&1
timeout 900 python tests/diag/skip_fuzz.py 300 5 > gpurun_out/skip_fuzz.txt 2>&1
# compute-sanitizer is closed on this GPU pool (late round 2): no sanitizer pass here
tail -5 gpurun_out/fuzz_wide.txt; tail -1 gpurun_out/skip_fuzz.txt
