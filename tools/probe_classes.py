"""Development aid: device time of a workload's narrow / wide problem classes
run separately (which class dominates the search)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from goldens import load, queries  # noqa: E402
from paper_2603_24595_b200.engine import compile_all  # noqa: E402
from paper_2603_24595_b200.native import Engine  # noqa: E402

eng = Engine(0)
for name in sys.argv[1:]:
    comp = compile_all(queries(load(name)))
    probs = [p for c, _ in comp if c for p in c.problems]
    for label, sel in (("narrow", [p for p in probs if p.narrow]),
                       ("wide", [p for p in probs if not p.narrow]), ("all", probs)):
        if not sel:
            continue
        eng.solve(sel, {"max_seconds": 600.0})
        st = eng.last_stats
        # per problem: the slowest single problems
        print(name, label, len(sel), "dev_ms %.1f boxes %d points %d" % (
            st["device_ms"], st["boxes"], st["points"]), flush=True)
    worst = []
    for i, p in enumerate(probs):
        eng.solve([p], {"max_seconds": 600.0})
        st = eng.last_stats
        worst.append((st["device_ms"], i, p.narrow, p.nvars, p.nregs, len(p.insns), st["boxes"]))
    worst.sort(reverse=True)
    for w in worst[:8]:
        print("  prob %d narrow=%s nv=%d nregs=%d ninsn=%d: %.1f ms, %d boxes" % (
            w[1], w[2], w[3], w[4], w[5], w[0], w[6]), flush=True)
