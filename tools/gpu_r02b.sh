mkdir -p gpurun_out
timeout 900 python tools/time_sites.py paged_attention_v2_long_b16 > gpurun_out/sites_v2long.jsonl 2> gpurun_out/sites_v2long.err
timeout 600 python tools/time_workloads.py paged_attention_v1 paged_attention_v1_long_b16 paged_attention_v2_long_b16 moe_align rotary_embedding > gpurun_out/times2.jsonl 2> gpurun_out/times2.err
timeout 600 python tools/bench_sort.py > gpurun_out/sort_bench.jsonl 2> gpurun_out/sort_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_k2sort.csv --profile-from-start off env MK_RACE_FORCE_SORT=1 python tools/profile_k2.py > gpurun_out/k2.json 2> gpurun_out/k2.err
timeout 600 env MK_RACE_FORCE_SORT=1 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_sort_pass -c 1 -o gpurun_out/prof_sort -f python tools/profile_k2.py > gpurun_out/ncu_full_sort.log 2>&1
ls -la gpurun_out
