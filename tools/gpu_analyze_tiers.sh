# GPU box: analyze() wall time with the B200 checking stage and device
# screening, single-query checks through both tiers vs the full tier only
mkdir -p gpurun_out
python - > gpurun_out/analyze_tiers.jsonl 2>&1 <<'PY'
import json, sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from refpath import add_reference, analyze_workload
assert add_reference()
from goldens import expected_findings, load
from paper_2603_24595_b200.detectors import install, uninstall
from paper_2603_24595_b200.engine import SiteChecker
chk = SiteChecker(device=0)
for w in ["rms_norm", "fused_add_rms_norm", "rotary_embedding", "moe_align_mixtral", "racy", "silu_and_mul", "paged_attention_v1"]:
    for tt in (True, False):
        chk.two_tier = tt
        ts = []
        for _ in range(4):
            prev = install(checker=chk, screening=True)
            t = time.perf_counter()
            try:
                got = analyze_workload(w)
            finally:
                uninstall(prev)
            ts.append((time.perf_counter() - t) * 1e3)
        print(json.dumps({"workload": w, "two_tier": tt, "ms": sorted(round(x, 1) for x in ts),
                          "findings_ok": got["findings"] == expected_findings(load(w))}), flush=True)
chk.close()
PY
