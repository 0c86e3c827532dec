# GPU box: K2 forced sort path per register cap of the compacting generator
mkdir -p gpurun_out
for m in ${MINBS:-0 3 4}; do
  MK_GC_MINB=$m bash tools/gpu_compact.sh; mv gpurun_out/compact.jsonl gpurun_out/compact_minb$m.jsonl
done
