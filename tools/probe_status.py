"""Development aid: per-problem verdicts of a workload decided as one batch
versus one problem at a time (the two must agree)."""
import os
import sys

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
    batch = eng.solve(probs, {"max_seconds": 600.0})
    bst = dict(eng.last_stats)
    diff = 0
    for i, p in enumerate(probs):
        solo = eng.solve([p], {"max_seconds": 600.0})[0]
        if solo != batch[i]:
            diff += 1
            print(name, "problem", i, "batch", batch[i], "solo", solo, flush=True)
    print(name, len(probs), "problems,", diff, "differ; batch stats", bst, flush=True)
