"""Experiment (GPU box): how many sites does the device decide from a
*light* compile (structural presolve only: no bound tightening, no
Fourier-Motzkin, no aggregation, no relaxation cuts, no dead-disjunct
pruning), within a short device budget?  Correctness is checked against the
goldens for every site the light pass decides."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from goldens import expected, load, queries, workloads  # noqa: E402
from paper_2603_24595_b200 import compiler as C  # noqa: E402
from paper_2603_24595_b200.engine import SiteChecker  # noqa: E402

P = C._Presolve
for n in ["_try_radix", "_try_quotient", "_try_aggregate", "_try_aggregate_ineq", "_try_fm",
          "_fbbt", "_try_relax", "_try_parallel"]:
    setattr(P, n, lambda self, lin, *a, **k: False)
_norm = P._normalize
P._normalize = lambda self, e, lin, ivl=None: _norm(self, e, lin, None)
C.OR_SPLIT = False


def main(budget_s, names):
    chk = SiteChecker(device=0, compile_workers=0, limits={"max_seconds": budget_s})
    for w in names:
        doc = load(w)
        qs = queries(doc)
        t0 = time.perf_counter()
        comp = []
        for q in qs:
            try:
                comp.append(C.compile_query(*q))
            except (C.CompileError, C.CapacityError) as exc:
                comp.append(None)
        tc = time.perf_counter() - t0
        ok = [(c, None) for c in comp if c is not None]
        idx = [i for i, c in enumerate(comp) if c is not None]
        t0 = time.perf_counter()
        # an absolute budget for the whole batch (not pooled per query)
        chk.limits = {"max_seconds": budget_s / max(len(ok), 1)}
        res = chk.decide(ok) if ok else []
        td = time.perf_counter() - t0
        host = dev = und = bad = 0
        for i, r in zip(idx, res):
            s = doc["sites"][i]
            v, wit = expected(s)
            cq = comp[i]
            if any(g.status == "unsat" for g in cq.groups):
                host += 1
                continue
            if r.status == "unknown":
                # not decided by the light tier (budget, or a float / give-up
                # component whose verdict the full presolve settles): the
                # product sends it to the second tier
                und += 1
                continue
            dev += 1
            if r.status != v or (v == "sat" and wit is not None and r.witness != wit):
                bad += 1
        print(json.dumps({"workload": w, "sites": len(qs), "compile_fail": len(qs) - len(idx),
                          "light_host_unsat": host, "device_decided": dev, "undecided": und,
                          "bad": bad, "compile_ms": round(tc * 1e3, 1),
                          "device_ms": round(td * 1e3, 1)}), flush=True)
    chk.close()


if __name__ == "__main__":
    main(float(sys.argv[1]), sys.argv[2:] or workloads())
