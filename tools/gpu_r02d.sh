mkdir -p gpurun_out
timeout 900 python tools/time_workloads.py paged_attention_v1_long_b8 paged_attention_v1_long_b16 paged_attention_v1_long_b32 paged_attention_v2_long_b16 paged_attention_v1 paged_attention_v2 moe_align rotary_embedding fused_add_rms_norm racy > gpurun_out/times3.jsonl 2> gpurun_out/times3.err
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
