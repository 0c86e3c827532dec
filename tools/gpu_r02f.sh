mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sort.py tests/test_race_sweep.py tests/test_replay.py -x -q -m gpu > gpurun_out/pytest_sort.log 2>&1; echo rc=$? >> gpurun_out/pytest_sort.log
timeout 600 python tools/bench_sort.py > gpurun_out/sort_bench.jsonl 2> gpurun_out/sort_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_k2sort.csv --profile-from-start off env MK_RACE_FORCE_SORT=1 python tools/profile_k2.py > gpurun_out/k2.json 2> gpurun_out/k2.err
timeout 600 python -c "
import sys, json, os; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
from bench import _race_sweep_line
from paper_2603_24595_b200.engine import SiteChecker
import argparse
chk = SiteChecker(device=0, compile_workers=0)
a = argparse.Namespace(race_tokens=262144)
print(json.dumps(_race_sweep_line(chk, a, {'hbm_gbs': 6540.2}, 'measured', 3.0e13)))
" > gpurun_out/k2line.json 2> gpurun_out/k2line.err
