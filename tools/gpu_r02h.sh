mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
MK_BENCH_ONE_DEVICE=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --analyze '' --access-tokens 0 --search '' > gpurun_out/bench_n2_onedevice.json 2> gpurun_out/bench_n2_onedevice.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
