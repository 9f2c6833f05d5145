#!/bin/bash
mkdir -p gpurun_out
for tool in ${TOOLS:-memcheck initcheck racecheck synccheck}; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit $?"; tail -3 gpurun_out/sanitize_$tool.log
done
