"""Development aid: end-to-end analyze() per workload with the B200
checking stage (GpuDetectors) vs the reference, split into checking-stage
time and front-end time (parser, DFS, branch screening)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from refpath import add_reference, analyze_workload  # noqa: E402

add_reference()
import minikernel.solver.interface as SI  # noqa: E402
from paper_2603_24595_b200.detectors import install, uninstall  # noqa: E402
from paper_2603_24595_b200.engine import SiteChecker  # noqa: E402

chk = SiteChecker(0)
orig = SI.Solver.check
for name in sys.argv[1:]:
    acc = {"screen_s": 0.0, "screen_calls": 0}

    def timed(self, assertions, bounds=None):
        t0 = time.perf_counter()
        try:
            return orig(self, assertions, bounds)
        finally:
            acc["screen_s"] += time.perf_counter() - t0
            acc["screen_calls"] += 1

    SI.Solver.check = timed
    prev = install(checker=chk, screening=os.environ.get("MK_SCREEN") == "1")
    c0 = chk.stats.compile_s + chk.stats.device_s + chk.stats.assemble_s
    t0 = time.perf_counter()
    try:
        doc = analyze_workload(name)
    finally:
        uninstall(prev)
        SI.Solver.check = orig
    wall = time.perf_counter() - t0
    c1 = chk.stats.compile_s + chk.stats.device_s + chk.stats.assemble_s
    print(json.dumps({"workload": name, "analyze_s": wall, "checking_s": c1 - c0,
                      "screen_fallbacks": sum(getattr(d, "screen_fallbacks", 0) for d in []),
                      "reference_solver_s": acc["screen_s"], "reference_solver_calls": acc["screen_calls"],
                      "findings": len(doc["findings"])}), flush=True)
chk.close()
