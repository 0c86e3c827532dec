"""Per-workload device timing (GPU box): compile on the host, upload the
problem set, run it resident a few times; prints one JSON line per
workload (compile ms, device ms, boxes, points, launches, parity)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from goldens import load, mismatches, queries, workloads  # noqa: E402
from paper_2603_24595_b200.engine import SiteChecker, compile_all  # noqa: E402


def main(names):
    # MK_LIB: an alternative build of libmk_b200.so (measurement of build variants)
    chk = SiteChecker(device=0, compile_workers=0, lib_path=os.environ.get("MK_LIB"))
    for name in names or workloads():
        doc = load(name)
        qs = queries(doc)
        t0 = time.perf_counter()
        comp = compile_all(qs)
        cms = 1e3 * (time.perf_counter() - t0)
        packed, offsets = chk.pack([c for c, _ in comp])
        res = chk.decide(comp, packed, offsets)
        bad = mismatches(doc, res)
        runs = []
        if packed.problems:
            rs = chk.engine.upload(packed)
            lim = dict(chk.limits)
            lim["max_seconds"] = 600.0
            runs = [rs.run(lim) for _ in range(3)]
            rs.free()
        out = {"workload": name, "sites": len(qs), "problems": len(packed.problems),
               "compile_ms": round(cms, 1), "parity_bad": len(bad)}
        if runs:
            r = runs[-1]
            out.update({"device_ms": [round(x["device_ms"], 3) for x in runs],
                        "boxes": r["boxes"], "points": r["points"], "launches": r["launches"],
                        "strategy": r.get("strategy")})
        print(json.dumps(out), flush=True)
    chk.close()


if __name__ == "__main__":
    main(sys.argv[1:])
