mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sort.py tests/test_replay.py -x -q -m gpu > gpurun_out/pytest_sort.log 2>&1; echo rc=$? >> gpurun_out/pytest_sort.log
timeout 300 python tools/bench_sort.py > gpurun_out/sort_bench.jsonl 2> gpurun_out/sort_bench.err
for v in "" _minb5 _minb6 _minb8; do
  MK_LIB=paper_2603_24595_b200/libmk_b200$v.so timeout 600 python tools/time_workloads.py moe_align paged_attention_v2_long_b16 paged_attention_v1 racy > gpurun_out/times_minb$v.jsonl 2>&1
done
