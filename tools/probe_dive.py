import os, sys
ROOT='/root/repo'
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'tests'))
from goldens import load, queries, mismatches
from paper_2603_24595_b200.engine import compile_all
from paper_2603_24595_b200.native import Engine, PackedSet
eng = Engine(0)
names = sys.argv[1:]
sets = {n: PackedSet([p for c, _ in compile_all(queries(load(n))) if c for p in c.problems]) for n in names}
for d in (4096,):
    for n in names:
        ms = []
        for rep in range(3):
            eng.solve_packed(sets[n], {"max_seconds": 600.0, "max_rounds": -d})
            ms.append(eng.last_stats["device_ms"])
        st = eng.last_stats
        print('dive', d, n, 'ms', ' '.join('%.2f' % x for x in ms), 'boxes', st['boxes'], 'steps', st['steps'], 'rounds', st['rounds'], 'launches', st['launches'], 'leaves', st['leaves'], 'points', st['points'], flush=True)
