"""Development aid: device statistics of single problems of a workload
(optionally with engine limits, e.g. chunk=-2 to disable the dive)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from goldens import load, queries  # noqa: E402
from paper_2603_24595_b200.engine import compile_all  # noqa: E402
from paper_2603_24595_b200.native import Engine  # noqa: E402

name = sys.argv[1]
want = [int(x) for x in sys.argv[2].split(",")]
extra = json.loads(sys.argv[3]) if len(sys.argv) > 3 else {}
probs = [p for c, _ in compile_all(queries(load(name))) if c for p in c.problems]
eng = Engine(0)
for i in want:
    lim = {"max_seconds": 60.0, **extra}
    r = eng.solve([probs[i]], lim)
    st = eng.last_stats
    print(i, r, {k: st[k] for k in ("boxes", "leaves", "points", "rounds", "device_ms", "launches", "steps")},
          flush=True)
