mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python tools/bench_sort.py > gpurun_out/sort_bench.jsonl 2> gpurun_out/sort_bench.err
python -m paper_2603_24595_b200 replay --kernel workloads/rms_norm/kernel.mk --context workloads/rms_norm/ctx.json > gpurun_out/replay_rms_norm.txt 2>&1
python -m paper_2603_24595_b200 replay --kernel workloads/paged_attention_v2_long_b16/kernel.mk --context workloads/paged_attention_v2_long_b16/ctx.json > gpurun_out/replay_pa_v2_long.txt 2>&1
