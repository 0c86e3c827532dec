mkdir -p gpurun_out
bash tools/gpu_profile_r02.sh config3 > gpurun_out/profile_r02.log 2>&1
bash tools/gpu_profile_r02.sh moe_align > gpurun_out/profile_r02_moe.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
