# GPU box: resident full-presolve step device time per search knob setting
# (MK_SPLIT_K split arity, MK_ADAPT_K shallow-stack widening), read by the
# engine at every call
mkdir -p gpurun_out
python - > gpurun_out/knobs.jsonl 2>&1 <<'PY'
import json, os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from paper_2603_24595_b200.engine import SiteChecker, compile_all
chk = SiteChecker(device=0, compile_workers=0)
sets = {}
for g in ["config3", "moe_align", "paged_attention_v2_long_b16", "paged_attention_v1", "racy"]:
    packed, _ = chk.pack([c for c, _ in compile_all(load_sites(entries(g))[1]) if c is not None])
    sets[g] = chk.engine.upload(packed)
for k in ["6", "8", "12", "16"]:
    for ad in ["0", "1"]:
        os.environ["MK_SPLIT_K"] = k
        os.environ["MK_ADAPT_K"] = ad
        for g, rs in sets.items():
            runs = [rs.run({"max_seconds": 600.0}) for _ in range(5)]
            print(json.dumps({"K": k, "adapt": ad, "group": g,
                              "ms": sorted(round(r["device_ms"], 2) for r in runs),
                              "boxes": runs[-1]["boxes"], "steps": runs[-1]["steps"]}), flush=True)
PY
