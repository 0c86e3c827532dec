mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sort.py tests/test_race_sweep.py tests/test_replay.py -x -q -m gpu > gpurun_out/pytest_sort.log 2>&1; echo rc=$? >> gpurun_out/pytest_sort.log
timeout 300 python tools/bench_sort.py > gpurun_out/sort_bench.jsonl 2> gpurun_out/sort_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_k2sortall.csv --profile-from-start off env MK_RACE_FORCE_SORT=1 MK_SORT_ALL_PASSES=1 python tools/profile_k2.py > gpurun_out/k2all.json 2> gpurun_out/k2all.err
