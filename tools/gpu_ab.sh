mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python tools/bench_configs.py C2 F1 > gpurun_out/cfg_two.jsonl 2>&1
KDE_DEBUG_ONE_STREAM=1 timeout 600 python tools/bench_configs.py C2 F1 > gpurun_out/cfg_one.jsonl 2>&1
tail -3 gpurun_out/pytest_gpu.txt
