# GPU box: where the e2e time of config3's check_queries goes (tier-1 / tier-2
# device calls, batches) for first-tier budget settings
mkdir -p gpurun_out
python - > gpurun_out/e2e_tiers.jsonl 2>&1 <<'PY'
import dataclasses, json, sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from paper_2603_24595_b200.engine import SiteChecker, BatchStats
qs = load_sites(entries("config3"))[1]
chk = SiteChecker(device=0)
import itertools
for t1, extra in itertools.product([(0.0005, 0.002, 0.01), (0.0002, 0.001, 0.005)],
                                   [{}, {"chunk": 65536}]):
    chk.TIER1_S = t1
    chk.TIER1_LIMITS = extra
    for _ in range(2):
        chk.check_queries(qs)
    walls = []
    for _ in range(6):
        chk.stats = BatchStats()
        t = time.perf_counter()
        res = chk.check_queries(qs)
        walls.append(round((time.perf_counter() - t) * 1e3, 1))
        st = dataclasses.asdict(chk.stats)
    st.pop("device", None)
    print(json.dumps({"tier1": t1, "extra": extra, "wall_ms": walls, "stats": st,
                      "verdicts": {v: sum(1 for r in res if r.status == v) for v in ("sat", "unsat", "unknown")}}), flush=True)
chk.TIER1_S = SiteChecker.TIER1_S
chk.trace = []
chk.check_queries(qs)
json.dump(chk.trace, open("gpurun_out/e2e_trace.json", "w"))
chk.close()
PY
