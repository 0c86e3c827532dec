# access replay (oracle rule): sort path and owner-table path launch lists
python tools/profile_access.py 16384 > gpurun_out/acc_step.json 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/acc_launches.csv python tools/profile_access.py 16384 > /dev/null 2>&1
python tools/summarize_k2.py gpurun_out/acc_launches.csv gpurun_out/acc_step.json gpurun_out/ncu_access_sort_summary.json mk_access_jit > /dev/null
python tools/profile_access.py 16384 fast > gpurun_out/acc_fast_step.json 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_lsu.sum,lts__t_sectors_op_atom.sum --clock-control none --csv --log-file gpurun_out/acc_fast_launches.csv python tools/profile_access.py 16384 fast > /dev/null 2>&1
python tools/summarize_k2.py gpurun_out/acc_fast_launches.csv gpurun_out/acc_fast_step.json gpurun_out/ncu_access_summary.json mk_access_jit > /dev/null
