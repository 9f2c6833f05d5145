#!/bin/bash
# A/B of software-exp columns in the 2048-tile Psi kernels (KDE_DEBUG_PSI_SW = m4*10 + m6): C4 time and
# parity against the C4 oracle golden (tools/bench_configs.py C4), one line per variant.
mkdir -p gpurun_out
: > gpurun_out/psi_sw_ab.jsonl
for v in ${VARIANTS:-0 1 2 10 20 30 11 21 22 31}; do
  echo "{\"variant\": $v}" >> gpurun_out/psi_sw_ab.jsonl
  KDE_DEBUG_PSI_SW=$v timeout 300 python tools/bench_configs.py C4 --reps 5 >> gpurun_out/psi_sw_ab.jsonl 2>> gpurun_out/psi_sw_ab.err
done
python - <<'PY'
import json
v=None
for l in open('gpurun_out/psi_sw_ab.jsonl'):
    d=json.loads(l)
    if 'variant' in d: v=d['variant']; continue
    print(v, round(d['wall_ms'],2), round(d['pair_ms'],2), d['parity']['rel_err'], d['clocks'].get('sm_mhz'))
PY
