mkdir -p gpurun_out
for v in "" _minb2 _minb3; do
python - > gpurun_out/minb$v.jsonl 2>&1 <<PY
import json, os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from paper_2603_24595_b200.engine import SiteChecker, compile_all
lib = "paper_2603_24595_b200/libmk_b200$v.so"
chk = SiteChecker(device=0, compile_workers=0, lib_path=lib)
for g in ["config3", "moe_align", "paged_attention_v2_long_b16", "racy"]:
    packed, _ = chk.pack([c for c, _ in compile_all(load_sites(entries(g))[1])])
    rs = chk.engine.upload(packed)
    runs = [rs.run({"max_seconds": 600.0}) for _ in range(5)]
    rs.free()
    print(json.dumps({"lib": lib, "group": g, "ms": sorted(round(r["device_ms"], 2) for r in runs)}), flush=True)
PY
done
