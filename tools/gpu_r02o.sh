mkdir -p gpurun_out
timeout 600 python tools/sweep_limits.py config3 > gpurun_out/sweep_c3.jsonl 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
