"""Development aid: device time per workload for alternative builds of the
engine library (occupancy / launch-bound variants)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from goldens import load, queries  # noqa: E402
from paper_2603_24595_b200.engine import compile_all  # noqa: E402
from paper_2603_24595_b200.native import Engine, PackedSet  # noqa: E402

libs = sys.argv[1].split(",")
names = sys.argv[2:]
sets = {}
for n in names:
    comp = compile_all(queries(load(n)))
    sets[n] = PackedSet([p for c, _ in comp if c for p in c.problems])
for lib in libs:
    eng = Engine(0, os.path.join(ROOT, "paper_2603_24595_b200", lib))
    for n in names:
        ms = []
        for rep in range(4):
            eng.solve_packed(sets[n], {"max_seconds": 600.0})
            ms.append(eng.last_stats["device_ms"])
        print(lib, n, "device_ms", " ".join("%.2f" % x for x in ms),
              "boxes %d" % eng.last_stats["boxes"], flush=True)
    eng.close()
