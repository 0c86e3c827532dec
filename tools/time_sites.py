"""Per-site device timing of one workload (GPU box): each device-decided
site's problems uploaded and run alone; prints the slowest sites."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from goldens import load, queries  # noqa: E402
from paper_2603_24595_b200.engine import SiteChecker, compile_all  # noqa: E402


def main(name, top=12):
    chk = SiteChecker(device=0, compile_workers=0)
    doc = load(name)
    comp = compile_all(queries(doc))
    out = []
    for i, (cq, _) in enumerate(comp):
        if cq is None or not cq.problems:
            continue
        packed, _ = chk.pack([cq])
        rs = chk.engine.upload(packed)
        lim = {"max_seconds": 600.0}
        runs = [rs.run(lim) for _ in range(2)]
        rs.free()
        s = doc["sites"][i]
        r = runs[-1]
        out.append({"site": i, "kind": s["site"], "line": s["line"], "verdict": s["verdict"],
                    "reason": s.get("reason"), "ms": r["device_ms"], "boxes": r["boxes"],
                    "points": r["points"],
                    "problems": [{"nvars": p.nvars, "nregs": p.nregs, "rows": len(p.rows),
                                  "narrow": p.narrow, "ninsn": len(p.insns),
                                  "vars": list(zip(p.var_names, map(str, p.lo), map(str, p.hi)))}
                                 for p in cq.problems]})
    out.sort(key=lambda r: -r["ms"])
    for r in out[:top]:
        print(json.dumps(r), flush=True)
    chk.close()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paged_attention_v2_long_b16")
