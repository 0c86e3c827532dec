mkdir -p gpurun_out
W=$(python -c "import sys; sys.path.insert(0,'tests'); from goldens import workloads; print(' '.join(w for w in workloads() if not w.startswith('topk')))")
for k in 16 8 12; do
  MK_SPLIT_K=$k timeout 900 python tools/time_workloads.py $W > gpurun_out/k$k.jsonl 2>&1
done
