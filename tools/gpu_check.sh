# GPU box session: sort tests, per-workload timings, GPU test suite, short bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 600 python -m pytest tests/test_sort.py -x -q > gpurun_out/pytest_sort.log 2>&1; echo rc=$? >> gpurun_out/pytest_sort.log
timeout 900 python tools/time_workloads.py paged_attention_v1_long_b8 paged_attention_v1_long_b16 paged_attention_v1_long_b32 paged_attention_v2_long_b16 paged_attention_v1 paged_attention_v2 copy_blocks silu_and_mul float_branch rms_norm_unknown_path rotary_embedding moe_align > gpurun_out/times.jsonl 2> gpurun_out/times.err
MK_HOST_FBBT=0 timeout 900 python tools/time_workloads.py paged_attention_v1_long_b16 paged_attention_v2_long_b16 paged_attention_v1 paged_attention_v2 moe_align rotary_embedding > gpurun_out/times_nofbbt.jsonl 2> gpurun_out/times_nofbbt.err
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
