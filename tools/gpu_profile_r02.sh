#!/bin/bash
# Round-2 profiling session (one GPU) for one workload group (default config3):
# ncu launch list of one resident step, then ncu --set full of the LONGEST
# k_search launch of that step (found from the launch list), the K2 sort path
# launch list and the INT32 microbenchmark counters.  Outputs in gpurun_out/.
mkdir -p gpurun_out
W=${1:-config3}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
export MK_REAL_STRATEGY=$(python -c "
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from paper_2603_24595_b200.engine import SiteChecker, compile_all
chk = SiteChecker(device=0, compile_workers=0)
packed, _ = chk.pack([c for c, _ in compile_all(load_sites(entries('$W'))[1])])
res = chk.engine.upload(packed)
print([res.run({'max_seconds': 600.0}) for _ in range(4)][-1]['strategy'])" 2>/dev/null | tail -1)
echo "real strategy: $MK_REAL_STRATEGY"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__thread_inst_executed.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_$W.csv \
    python tools/profile_step.py $W > gpurun_out/step_$W.json 2> gpurun_out/step_$W.err
SKIP=$(python - <<PY
import csv
rows = list(csv.reader(open("gpurun_out/launches_$W.csv")))
hdr = None; t = {}
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    if "k_search" in d["Kernel Name"] and d["Metric Name"] == "gpu__time_duration.sum":
        t[int(d["ID"])] = float(d["Metric Value"].replace(",", ""))
ids = sorted(t)
print(ids.index(max(ids, key=lambda i: t[i])) if ids else 0)
PY
)
echo "longest k_search launch: #$SKIP"
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_search -s $SKIP -c 1 \
    -o gpurun_out/prof_$W -f python tools/profile_step.py $W > gpurun_out/ncu_full_$W.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_k2sort.csv --profile-from-start off env MK_RACE_FORCE_SORT=1 python tools/profile_k2.py \
    > gpurun_out/k2.json 2> gpurun_out/k2.err
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__thread_inst_executed.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none --csv --log-file gpurun_out/int_peak.csv -k regex:k_int_peak \
    python -c "
import sys; sys.path.insert(0, '.')
from paper_2603_24595_b200.native import Engine
e = Engine(0); print(e.int_peak()); e.close()" > gpurun_out/int_peak.json 2>&1
ls -la gpurun_out
