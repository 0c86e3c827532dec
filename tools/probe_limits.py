"""Development aid: resident step time of a workload under engine limit
variants (e.g. chunk=-1: no pre-split, roots straight to the persistent
search)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from goldens import load, mismatches, queries  # noqa: E402
from paper_2603_24595_b200.engine import SiteChecker, compile_all  # noqa: E402

name = sys.argv[1]
chk = SiteChecker(device=0, compile_workers=0)
doc = load(name)
comp = compile_all(queries(doc))
packed, offsets = chk.pack([c for c, _ in comp])
res = chk.engine.upload(packed)
for spec in sys.argv[2:]:
    lim = dict(chk.limits)
    lim["max_seconds"] = 600.0
    lim.update(json.loads(spec))
    for _ in range(3):
        res.run(lim)
    runs = [res.run(lim) for _ in range(10)]
    ms = sorted(r["device_ms"] for r in runs)
    print(spec, "device_ms median %.3f min %.3f" % (ms[5], ms[0]),
          {k: runs[-1][k] for k in ("boxes", "points", "rounds", "launches", "steps")}, flush=True)
saved = dict(chk.limits)
for spec in sys.argv[2:]:
    chk.limits = dict(saved, **json.loads(spec))
    bad = mismatches(doc, chk.decide(comp, packed, offsets))
    print(spec, "parity", "ok" if not bad else bad[:5])
res.free()
chk.close()
