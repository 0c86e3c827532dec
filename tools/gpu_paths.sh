# GPU box: device time of the resident search step per k_search code-path
# variant (A: no "small" path, B: no shared-register path, C: neither);
# VARIANTS="base _X ..." picks the libraries (libmk_b200$v.so)
mkdir -p gpurun_out
for v in ${VARIANTS:-base _A _B _C}; do
[ "$v" = base ] && v=""
python - > gpurun_out/paths$v.jsonl 2>&1 <<PY
import json, os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from paper_2603_24595_b200.engine import SiteChecker, compile_all
lib = "paper_2603_24595_b200/libmk_b200$v.so"
chk = SiteChecker(device=0, compile_workers=0, lib_path=lib)
for g in ["config3", "moe_align", "paged_attention_v2_long_b16", "racy", "rms_norm", "rotary_embedding"]:
    for light in (True, False):
        packed, _ = chk.pack([c for c, _ in compile_all(load_sites(entries(g))[1], light=light) if c is not None])
        rs = chk.engine.upload(packed)
        runs = [rs.run({"max_seconds": 0.5 if light else 600.0}) for _ in range(5)]
        st = {int(k): int(v) for k, v in zip(*__import__("numpy").unique(rs.status[:len(packed.problems)], return_counts=True))}
        rs.free()
        print(json.dumps({"lib": lib, "group": g, "light": light, "status": st, "ms": sorted(round(r["device_ms"], 2) for r in runs)}), flush=True)
PY
done
