mkdir -p gpurun_out
W="config3 moe_align paged_attention_v2_long_b16 racy fused_add_rms_norm paged_attention_v1 rotary_embedding"
python - <<'PY' > gpurun_out/adapt.jsonl 2>&1
import json, os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from goldens import mismatches
from paper_2603_24595_b200.engine import SiteChecker, compile_all
chk = SiteChecker(device=0, compile_workers=0)
for g in ["config3", "moe_align", "paged_attention_v2_long_b16", "racy", "fused_add_rms_norm", "paged_attention_v1", "rotary_embedding", "paged_attention_v2", "copy_blocks"]:
    docs, qs, recs = load_sites(entries(g))
    comp = compile_all(qs)
    for adapt in ("0", "1"):
        os.environ["MK_ADAPT_K"] = adapt
        res = chk.decide(comp)
        bad = mismatches({"sites": recs}, res)
        packed, _ = chk.pack([c for c, _ in comp])
        rs = chk.engine.upload(packed)
        runs = [rs.run({"max_seconds": 600.0}) for _ in range(4)]
        rs.free()
        print(json.dumps({"group": g, "adapt": adapt, "bad": len(bad), "ms": sorted(round(r["device_ms"], 2) for r in runs),
                          "boxes": min(r["boxes"] for r in runs), "steps": min(r["steps"] for r in runs)}), flush=True)
PY
