# GPU box: fixed cost of one engine call (tiny problem sets), wall vs device
mkdir -p gpurun_out
python - > gpurun_out/call_overhead.txt 2>&1 <<'PY'
import sys, time, json
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from goldens import load, queries
from paper_2603_24595_b200.engine import SiteChecker, compile_all
chk = SiteChecker(device=0, compile_workers=0)
doc = load("racy"); qs = queries(doc)
comp = [c for c in compile_all(qs) if c[0] is not None and c[0].problems]
for n in (1, 4):
    sub = comp[:n]
    for budget in (None, 0.002):
        for _ in range(5): chk.decide(sub, budget_s=budget)
        ts, dev = [], []
        for _ in range(30):
            t = time.perf_counter(); chk.decide(sub, budget_s=budget); ts.append(time.perf_counter() - t)
            dev.append(chk.engine.last_stats["device_ms"])
        ts.sort(); dev.sort()
        print(json.dumps({"queries": n, "budget": budget, "wall_ms_median": round(ts[15] * 1e3, 3),
                          "device_ms_median": round(dev[15], 3), "launches": chk.engine.last_stats["launches"],
                          "strategy": chk.engine.last_stats["strategy"]}))
PY
