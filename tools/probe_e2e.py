"""Development aid: split of one public-API call (SiteChecker.check_queries)
into compile / pack / device / assemble."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from goldens import load, queries  # noqa: E402
from paper_2603_24595_b200.engine import SiteChecker  # noqa: E402

chk = SiteChecker(0)
for name in sys.argv[1:]:
    qs = queries(load(name))
    for rep in range(4):
        t0 = time.perf_counter()
        comp = chk.compile(qs)
        t1 = time.perf_counter()
        packed, offs = chk.pack([c for c, _ in comp])
        t2 = time.perf_counter()
        res = chk.decide(comp, packed, offs)
        t3 = time.perf_counter()
        st = chk.engine.last_stats
    per = sorted((c.compile_s for c, _ in comp if c is not None), reverse=True)
    print(name, "compile %.1f ms (sum %.1f ms, max %.2f ms, n %d, workers %d), pack %.1f ms, "
          "decide %.1f ms (device %.1f ms, call %.1f ms)" % (
              1e3 * (t1 - t0), 1e3 * sum(per), 1e3 * per[0], len(per), chk.compile_workers,
              1e3 * (t2 - t1), 1e3 * (t3 - t2), st["device_ms"], 1e3 * st["seconds"]), flush=True)
chk.close()
