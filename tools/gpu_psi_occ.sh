#!/bin/bash
# A/B: Psi kernels at 4 CTAs/SM (64 regs) vs 3 CTAs/SM (80 regs).  Output under gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_occ4.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_occ4.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 2 -c 1 \
    -o gpurun_out/prof_psi6_occ4 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_occ4.log 2>&1
sed -i 's/MINB = 1024 \/ NT_;/MINB = 768 \/ NT_;/' paper_1505_01998_b200/csrc/kde_pair.cuh
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_occ3.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_occ3.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 2 -c 1 \
    -o gpurun_out/prof_psi6_occ3 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_occ3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 3 -c 1 \
    -o gpurun_out/prof_psi4_occ3 -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_occ3b.log 2>&1
grep -h -o '"ms_per_step": [0-9.]*' gpurun_out/bench_occ4.json gpurun_out/bench_occ3.json
