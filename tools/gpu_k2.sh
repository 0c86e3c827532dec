MK_RACE_FORCE_SORT=1 python tools/profile_k2.py > gpurun_out/k2_sort_step.json 2>&1
MK_RACE_FORCE_SORT=1 timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/k2_sort_launches.csv python tools/profile_k2.py > /dev/null 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
