"""Development aid: which store sites' K2 keys arrive out of order (the
radix-sort path), and their sizes."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_race_sweep import _cases
from paper_2603_24595_b200.native import Engine
eng = Engine(0)
for name, i, launch, expect, prog in _cases():
    r = eng.race_sweep(prog)
    if not r["sorted"]:
        print(name, i, prog.instances, r["tuples"], r["sort_bits"], {k: launch.get(k) for k in ("BS", "SL", "TC", "gridDim.x", "blockDim.x")}, prog.problem.var_names, flush=True)
