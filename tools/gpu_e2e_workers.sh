# GPU box: config3 check_queries wall time per compile-pool size
mkdir -p gpurun_out
python - > gpurun_out/e2e_workers.jsonl 2>&1 <<'PY'
import json, os, sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from paper_2603_24595_b200.engine import SiteChecker
qs = load_sites(entries("config3"))[1]
for w in (11, 13, 15, 16):
    chk = SiteChecker(device=0, compile_workers=w)
    for _ in range(3):
        chk.check_queries(qs)
    walls = []
    for _ in range(8):
        t = time.perf_counter(); chk.check_queries(qs); walls.append(round((time.perf_counter() - t) * 1e3, 1))
    walls.sort()
    print(json.dumps({"workers": w, "wall_ms": walls, "median": walls[4], "cpus": os.cpu_count()}), flush=True)
    chk.close()
PY
