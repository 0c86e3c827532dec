# GPU box: config3's first tier (light problems, 20 ms budget) per task-grab
# size: device time (budget overrun) and decided counts
mkdir -p gpurun_out
python - > gpurun_out/tier1_group.jsonl 2>&1 <<'PY'
import json, os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from paper_2603_24595_b200.engine import SiteChecker, compile_all
chk = SiteChecker(device=0, compile_workers=0)
light = [c for c, _ in compile_all(load_sites(entries("config3"))[1], light=True) if c is not None]
packed, _ = chk.pack(light)
rs = chk.engine.upload(packed)
import numpy as np
for g in ["16"]:
    os.environ["MK_TASK_GROUP"] = g
    for budget, chunk in ((0.02, 0), (0.05, 0), (0.02, -2), (0.05, -2), (0.05, 1024)):
        runs = [rs.run({"max_seconds": budget, "chunk": chunk}) for _ in range(5)]
        st = np.unique(rs.status[:len(packed.problems)], return_counts=True)
        print(json.dumps({"group": g, "budget_s": budget, "chunk": chunk, "bb_ms": round(runs[-1]["bb_ms"], 2), "leaf_ms": round(runs[-1]["leaf_ms"], 2), "seconds": round(runs[-1]["seconds"], 4), "launches": runs[-1]["launches"], "ms": sorted(round(r["device_ms"], 2) for r in runs),
                          "points": runs[-1]["points"], "boxes": runs[-1]["boxes"], "rounds": runs[-1]["rounds"],
                          "status": {int(a): int(b) for a, b in zip(*st)}}), flush=True)
PY
