mkdir -p gpurun_out
MK_TRACE_RUN=1 python - > gpurun_out/trace_run.txt 2>&1 <<'PY'
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from paper_2603_24595_b200.engine import SiteChecker, compile_all
chk = SiteChecker(device=0, compile_workers=0)
light = [c for c, _ in compile_all(load_sites(entries("config3"))[1], light=True) if c is not None]
packed, _ = chk.pack(light)
rs = chk.engine.upload(packed)
for budget in (0.05, 0.05, 0.02):
    r = rs.run({"max_seconds": budget})
    print("RUN", budget, r["device_ms"], r["seconds"], file=sys.stderr, flush=True)
PY
