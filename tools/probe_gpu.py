"""Quick GPU probe: decide every golden workload in one batch and per query,
print timings and device statistics (development aid)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from goldens import load, mismatches, queries, workloads  # noqa: E402
from paper_2603_24595_b200.engine import SiteChecker, compile_all  # noqa: E402

chk = SiteChecker(device=0)
out = {}
for name in workloads():
    doc = load(name)
    qs = queries(doc)
    t0 = time.perf_counter()
    comp = compile_all(qs)
    t1 = time.perf_counter()
    packed, offs = chk.pack([c for c, _ in comp])
    for rep in range(2):
        t2 = time.perf_counter()
        res = chk.decide(comp, packed, offs)
        t3 = time.perf_counter()
    bad = mismatches(doc, res)
    st = dict(chk.engine.last_stats)
    t4 = time.perf_counter()
    res1 = [chk.check(*q) for q in qs] if len(qs) <= 64 else res
    t5 = time.perf_counter()
    bad1 = mismatches(doc, res1)
    out[name] = dict(sites=len(qs), compile_s=t1 - t0, batch_s=t3 - t2, single_s=t5 - t4,
                     ref_s=doc["reference_wall_s"], bad=len(bad), bad_single=len(bad1),
                     stats=st)
    print(name, json.dumps(out[name]), flush=True)
    if bad:
        print("  first mismatches:", bad[:5])
        print("  unknown:", sum(1 for r in res if r.status == "unknown"))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "probe.json"), "w"), indent=1)
