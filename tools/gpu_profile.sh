#!/bin/bash
# GPU-box session: bench line, reference arm, ncu launch list, ncu full capture
# of the persistent search kernel.  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
W=${1:-rotary_embedding}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 600 python bench.py --workload $W --steps 10 --warmup 3 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
timeout 300 python bench.py --impl reference --workload $W --steps 3 --warmup 1 > gpurun_out/bench_ref_$W.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$W.csv python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_search -s 3 -c 1 \
    -o gpurun_out/prof_$W -f python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$W.log 2>&1
ls -la gpurun_out
