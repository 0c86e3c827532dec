mkdir -p gpurun_out
W="paged_attention_v1 paged_attention_v1_long_b16 paged_attention_v2_long_b16 moe_align rotary_embedding fused_add_rms_norm racy"
timeout 600 python tools/time_workloads.py $W > gpurun_out/rs_default.jsonl 2>&1
MK_ROOT_SWEEPS=0 timeout 600 python tools/time_workloads.py $W > gpurun_out/rs_off.jsonl 2>&1
MK_HOST_FBBT=0 timeout 900 python tools/time_workloads.py $W > gpurun_out/rs_nohost.jsonl 2>&1
MK_HOST_FBBT=0 MK_ROOT_SWEEPS=512 timeout 900 python tools/time_workloads.py $W > gpurun_out/rs_nohost512.jsonl 2>&1
