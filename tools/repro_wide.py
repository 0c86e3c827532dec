"""Development aid: run one workload's wide (or narrow) problems alone."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from goldens import load, queries  # noqa: E402
from paper_2603_24595_b200.engine import compile_all  # noqa: E402
from paper_2603_24595_b200.native import Engine  # noqa: E402

name, cls = sys.argv[1], sys.argv[2]
secs = float(sys.argv[3]) if len(sys.argv) > 3 else 30.0
comp = compile_all(queries(load(name)))
probs = [p for c, _ in comp if c for p in c.problems]
sel = [p for p in probs if p.narrow == (cls == "narrow")]
if len(sys.argv) > 4:
    sel = [sel[int(i)] for i in sys.argv[4].split(",")]
print(len(sel), "problems", [(p.nvars, p.nregs) for p in sel][:40], flush=True)
eng = Engine(0)
res = eng.solve(sel, {"max_seconds": secs})
print([r[0] for r in res], eng.last_stats, flush=True)
