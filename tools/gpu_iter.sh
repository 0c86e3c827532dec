# GPU box: one k_search iteration check -- GPU tests, resident-step device
# times of the in-tree library against the variants named in VARIANTS, and
# the ncu profile of config3's longest k_search launch
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
bash tools/gpu_paths.sh
[ -n "$PROFILE" ] && bash tools/gpu_profile_r02.sh config3 > gpurun_out/profile_r02.log 2>&1
true
