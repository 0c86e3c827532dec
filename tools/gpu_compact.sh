# GPU box: config 1's K2 sort path (MK_RACE_FORCE_SORT) per compaction tile
# build (libmk_b200$v.so): generation / compaction+order / scan times
mkdir -p gpurun_out
for v in ${VARIANTS:-base}; do
[ "$v" = base ] && v=""
MK_RACE_FORCE_SORT=1 python - > gpurun_out/compact$v.jsonl 2>&1 <<PY
import json, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from goldens import load, queries
from paper_2603_24595_b200 import race
from paper_2603_24595_b200.engine import SiteChecker
chk = SiteChecker(device=0, compile_workers=0, lib_path="paper_2603_24595_b200/libmk_b200$v.so")
doc = load("rms_norm"); qs = queries(doc); T = 262144
launch = {"BS": 1, "SL": T, "TC": T, "blockDim.x": 1024, "blockDim.y": 1, "blockDim.z": 1,
          "gridDim.x": T, "gridDim.y": 1, "gridDim.z": 1}
progs = [race.race_program(a, o, launch) for s, (a, o) in zip(doc["sites"], qs)
         if s["site"] == "store_site" and s["line"] == 20]
prog = max(progs, key=lambda p: p.instances)
for _ in range(2):
    chk.engine.race_sweep(prog)
rs = [chk.engine.race_sweep(prog) for _ in range(7)]
tot = sorted(r["gen_ms"] + r["sort_ms"] + r["scan_ms"] for r in rs)
print(json.dumps({"lib": "$v", "total_ms": tot, "gen": sorted(r["gen_ms"] for r in rs)[3],
                  "sort": sorted(r["sort_ms"] for r in rs)[3], "scan": sorted(r["scan_ms"] for r in rs)[3],
                  "tuples": rs[0]["tuples"], "conflicts": rs[0]["conflicts"]}))
PY
done
