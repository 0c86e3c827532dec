"""Search-parameter sweep (GPU box): resident device time of a workload
group under split arity K and leaf volume variations (measurement only)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from bench import entries, load_sites  # noqa: E402
from paper_2603_24595_b200.engine import SiteChecker, compile_all  # noqa: E402


def main(groups):
    chk = SiteChecker(device=0, compile_workers=0)
    for g in groups:
        packed, _ = chk.pack([c for c, _ in compile_all(load_sites(entries(g))[1])])
        rs = chk.engine.upload(packed)
        for k in (8, 12, 16, 32):
            for leaf in (1024, 4096, 16384):
                lim = {"max_seconds": 600.0, "split_k": k, "leaf_volume": leaf}
                runs = [rs.run(lim) for _ in range(4)]
                print(json.dumps({"group": g, "K": k, "leaf": leaf,
                                  "ms": sorted(round(r["device_ms"], 2) for r in runs),
                                  "boxes": [r["boxes"] for r in runs]}), flush=True)
        rs.free()
    chk.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["moe_align", "config3"])
