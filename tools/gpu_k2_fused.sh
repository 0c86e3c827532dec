# GPU box: K2 sort path with the compacting generator (tile sizes via
# MK_GC_ITEMS) against dense generation + separate compaction
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_race_sweep.py tests/test_sort.py tests/test_replay.py tests/test_shard.py -m gpu -x -q > gpurun_out/pytest_k2.log 2>&1; echo rc=$? >> gpurun_out/pytest_k2.log
for it in 8 16 32 64; do
  MK_GC_ITEMS=$it bash tools/gpu_compact.sh; mv gpurun_out/compact.jsonl gpurun_out/compact_fused_$it.jsonl
done
MK_RACE_SEPARATE_COMPACT=1 bash tools/gpu_compact.sh; mv gpurun_out/compact.jsonl gpurun_out/compact_separate.jsonl
