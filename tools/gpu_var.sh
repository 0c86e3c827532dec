mkdir -p gpurun_out
python - > gpurun_out/var.jsonl 2>&1 <<'PY'
import json, os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from paper_2603_24595_b200.engine import SiteChecker, compile_all
chk = SiteChecker(device=0, compile_workers=0)
packed, _ = chk.pack([c for c, _ in compile_all(load_sites(entries("config3"))[1])])
rs = chk.engine.upload(packed)
for mode in ("default", "noprobe"):
    if mode == "noprobe":
        os.environ["MK_NO_PROBE"] = "1"
    for i in range(30):
        r = rs.run({"max_seconds": 600.0})
        print(json.dumps({"mode": mode, "ms": round(r["device_ms"], 2), "strategy": r["strategy"], "boxes": r["boxes"],
                          "rounds": r["rounds"], "launches": r["launches"], "bb_ms": round(r["bb_ms"], 2)}), flush=True)
rs.free()
PY
