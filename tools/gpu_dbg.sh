mkdir -p gpurun_out
timeout 600 python tools/lscv_variants.py 0 3 5 6 7 8 > gpurun_out/lscv_variants2.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python tools/bench_configs.py C3 C5P > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
cat gpurun_out/lscv_variants2.jsonl; tail -5 gpurun_out/pytest_gpu.txt; cat gpurun_out/bench.json gpurun_out/configs.jsonl
