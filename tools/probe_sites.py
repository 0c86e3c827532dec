"""Per-query GPU timing for one workload (development aid)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from goldens import load, queries
from paper_2603_24595_b200.engine import SiteChecker
chk = SiteChecker(device=0)
doc = load(sys.argv[1])
for i, q in enumerate(queries(doc)):
    t = time.perf_counter()
    r = chk.check(*q)
    dt = time.perf_counter() - t
    st = chk.engine.last_stats or {}
    print(i, doc["sites"][i]["site"], r.status, doc["sites"][i]["verdict"], f"{dt*1000:.1f}ms",
          {k: st.get(k) for k in ("rounds", "boxes", "leaves", "points", "bb_ms")}, flush=True)
