# GPU box: the caller's process during config3's check_queries: time spent
# pickling jobs, unpickling results, packing, in device calls and assembling
# (monkeypatched timers, accumulated over all threads)
mkdir -p gpurun_out
python - > gpurun_out/e2e_profile.txt 2>&1 <<'PY'
import collections, json, pickle, sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from paper_2603_24595_b200 import engine as E
from paper_2603_24595_b200.compiler import CompiledQuery
qs = load_sites(entries("config3"))[1]
chk = E.SiteChecker(device=0)
acc = collections.Counter()
def timed(name, f):
    def w(*a, **k):
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            acc[name] += time.perf_counter() - t
    return w
_dumps, _loads = pickle.dumps, pickle.loads
pickle.dumps = timed("pickle.dumps", _dumps)
pickle.loads = timed("pickle.loads", _loads)
E.SiteChecker.pack = timed("pack", E.SiteChecker.pack)
E.SiteChecker.decide = timed("decide (total)", E.SiteChecker.decide)
CompiledQuery.assemble = timed("assemble", CompiledQuery.assemble)
from paper_2603_24595_b200 import native as N
N.Engine.solve_packed = timed("engine.solve_packed", N.Engine.solve_packed)
for _ in range(3):
    chk.check_queries(qs)
acc.clear()
walls = []
for _ in range(5):
    t = time.perf_counter(); chk.check_queries(qs); walls.append(time.perf_counter() - t)
print(json.dumps({"wall_ms": sorted(round(w * 1e3, 1) for w in walls),
                  "per_call_ms": {k: round(v * 1e3 / 5, 1) for k, v in acc.most_common()}}, indent=1))
chk.close()
PY
