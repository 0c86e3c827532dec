"""Experiment (GPU box): how many sites the first tier decides per golden
workload -- the product's light compile (``compile_query(light=True)``:
structural presolve only) searched on the device under the first tier's
limits and batch budget (``SiteChecker.TIER1_S`` / ``TIER1_LIMITS``), one
batch per workload.  Every decided site is checked against the goldens."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from goldens import expected, load, queries, workloads  # noqa: E402
from paper_2603_24595_b200.engine import SiteChecker, _compile_one  # noqa: E402


def main(names):
    chk = SiteChecker(device=0, compile_workers=0)
    for w in names:
        doc = load(w)
        qs = queries(doc)
        t0 = time.perf_counter()
        comp = [_compile_one((a, o, True)) for a, o in qs]
        tc = time.perf_counter() - t0
        idx = [i for i, (c, _) in enumerate(comp) if c is not None]
        t0 = time.perf_counter()
        res = chk.decide([comp[i] for i in idx], budget_s=chk.tier1_budget(len(idx))) if idx else []
        td = time.perf_counter() - t0
        host = dev = und = bad = 0
        for i, r in zip(idx, res):
            v, wit = expected(doc["sites"][i])
            if any(g.status == "unsat" for g in comp[i][0].groups):
                host += 1                      # constant folding in the light compile
                if r.status != "unsat" or v != "unsat":
                    bad += 1
                continue
            if r.status not in ("sat", "unsat"):
                und += 1                       # left to the second tier
                continue
            dev += 1
            if r.status != v or (v == "sat" and wit is not None and r.witness != wit):
                bad += 1
        print(json.dumps({"workload": w, "sites": len(qs), "light_failed": len(qs) - len(idx),
                          "light_host_unsat": host, "device_decided": dev, "undecided": und,
                          "bad": bad, "compile_ms": round(tc * 1e3, 1),
                          "device_ms": round(td * 1e3, 1)}), flush=True)
    chk.close()


if __name__ == "__main__":
    main(sys.argv[1:] or workloads())
