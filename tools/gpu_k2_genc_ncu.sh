# GPU box: ncu --set full of the compacting K2 generator (config 1 store,
# forced sort path)
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:mk_race_genc_jit -c 1 \
    -o gpurun_out/prof_k2_genc -f env MK_RACE_FORCE_SORT=1 python tools/profile_k2.py > gpurun_out/k2_genc.log 2>&1
