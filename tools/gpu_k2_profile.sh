# GPU box: ncu launch lists of config 1's K2 sort path (forced; and with
# every radix pass forced) with per-kernel time and DRAM bytes
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_k2sort.csv --profile-from-start off env MK_RACE_FORCE_SORT=1 python tools/profile_k2.py \
    > gpurun_out/k2.json 2> gpurun_out/k2.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_k2sortall.csv --profile-from-start off env MK_RACE_FORCE_SORT=1 MK_SORT_ALL_PASSES=1 python tools/profile_k2.py \
    > gpurun_out/k2all.json 2> gpurun_out/k2all.err
