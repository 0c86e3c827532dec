mkdir -p gpurun_out
export MK_REAL_STRATEGY=0
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_search -s 5 -c 1 -o gpurun_out/prof_moe_align -f python tools/profile_step.py moe_align > gpurun_out/ncu_full_moe_align.log 2>&1
timeout 900 python tools/time_sites.py paged_attention_v2_long_b16 > gpurun_out/sites_v2long_after.jsonl 2> gpurun_out/sites_v2long_after.err
