#!/bin/bash
# GPU-box session for one workload: bench line, reference arm, ncu launch
# list of one resident step (per-kernel time + thread instructions), ncu full
# capture of the persistent search kernel.  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
W=${1:-rotary_embedding}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 600 python bench.py --workload $W --steps 10 --warmup 3 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
timeout 600 python bench.py --impl reference --workload $W --steps 3 --warmup 1 > gpurun_out/bench_ref_$W.json 2>&1
export MK_REAL_STRATEGY=$(python -c "
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from goldens import load, queries
from paper_2603_24595_b200.engine import SiteChecker, compile_all
chk = SiteChecker(device=0, compile_workers=0)
packed, _ = chk.pack([c for c, _ in compile_all(queries(load('$W')))])
res = chk.engine.upload(packed)
print([res.run({'max_seconds': 600.0}) for _ in range(4)][-1]['strategy'])" 2>/dev/null | tail -1)
echo "real strategy: $MK_REAL_STRATEGY"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__thread_inst_executed.sum,smsp__inst_executed.sum \
    --clock-control none --csv --log-file gpurun_out/launches_$W.csv \
    python tools/profile_step.py $W > gpurun_out/step_$W.json 2> gpurun_out/step_$W.err
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_search -s 2 -c 2 \
    -o gpurun_out/prof_$W -f python tools/profile_step.py $W > gpurun_out/ncu_full_$W.log 2>&1
ls -la gpurun_out
