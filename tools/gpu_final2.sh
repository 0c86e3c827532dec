mkdir -p gpurun_out
timeout 700 python tools/light_experiment.py 0.02 > gpurun_out/light_tier.jsonl 2>&1
bash tools/gpu_bench.sh
