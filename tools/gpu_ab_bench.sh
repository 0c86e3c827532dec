# GPU box: the headline bench line (no side lines) for the in-tree library and
# for libmk_b200$V.so swapped in (box copy only), alternating twice
mkdir -p gpurun_out
cp paper_2603_24595_b200/libmk_b200.so /tmp/libmk_base.so
for round in 1 2; do
  for v in base $V; do
    if [ "$v" = base ]; then cp /tmp/libmk_base.so paper_2603_24595_b200/libmk_b200.so;
    else cp paper_2603_24595_b200/libmk_b200$v.so paper_2603_24595_b200/libmk_b200.so; fi
    timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --analyze "" --search "" \
      --access-tokens 0 --race-tokens 0 > gpurun_out/ab_${v}_$round.json 2> gpurun_out/ab_${v}_$round.err
  done
done
cp /tmp/libmk_base.so paper_2603_24595_b200/libmk_b200.so
