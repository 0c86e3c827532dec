# GPU box: config3's first tier (light problems) under the first tier's
# limits (10 ms budget, no probe) per split arity: undecided counts and time
mkdir -p gpurun_out
python - > gpurun_out/tier1_k.jsonl 2>&1 <<'PY'
import json, os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from paper_2603_24595_b200.engine import SiteChecker, compile_all
import numpy as np
chk = SiteChecker(device=0, compile_workers=0)
light = [c for c, _ in compile_all(load_sites(entries("config3"))[1], light=True) if c is not None]
packed, _ = chk.pack(light)
rs = chk.engine.upload(packed)
for k in ["6", "8", "12", "16"]:
    os.environ["MK_SPLIT_K"] = k
    for budget in (0.01, 0.02):
        und = []
        ms = []
        for _ in range(5):
            r = rs.run({"max_seconds": budget, "chunk": 65536})
            ms.append(round(r["device_ms"], 2))
            und.append(int((rs.status[:len(packed.problems)] == 2).sum()))
        print(json.dumps({"K": k, "budget_s": budget, "ms": sorted(ms), "undecided": sorted(und)}), flush=True)
PY
