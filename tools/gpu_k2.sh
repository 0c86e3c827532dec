# K2 fused race pass: launch list (per-kernel time, DRAM bytes, SASS thread
# instructions) and one --set full capture of the fused kernel
python tools/profile_k2.py > gpurun_out/k2_step.json 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum --clock-control none --csv --log-file gpurun_out/k2_launches.csv python tools/profile_k2.py > /dev/null 2>&1
python tools/summarize_k2.py gpurun_out/k2_launches.csv gpurun_out/k2_step.json gpurun_out/ncu_k2_summary.json > /dev/null
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:mk_race_fused_jit -c 1 -o gpurun_out/prof_k2 -f python tools/profile_k2.py > gpurun_out/ncu_full_k2.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none -k regex:mk_access_jit -c 2 -o gpurun_out/prof_access -f python tools/profile_access.py 16384 fast > gpurun_out/ncu_full_access.log 2>&1
