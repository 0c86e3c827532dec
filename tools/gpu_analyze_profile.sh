# GPU box: cProfile of analyze() on one workload with the B200 checking stage
# and device screening installed (where the time-to-verdict goes)
mkdir -p gpurun_out
python - > gpurun_out/analyze_profile.txt 2>&1 <<'PY'
import cProfile, pstats, sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from refpath import add_reference, analyze_workload
assert add_reference()
from paper_2603_24595_b200.detectors import install, uninstall
from paper_2603_24595_b200.engine import SiteChecker
chk = SiteChecker(device=0)
for w in ["rms_norm"]:
    for _ in range(2):
        prev = install(checker=chk, screening=True); analyze_workload(w); uninstall(prev)
    prev = install(checker=chk, screening=True)
    t = time.perf_counter(); analyze_workload(w); print(w, "wall ms", (time.perf_counter() - t) * 1e3)
    pr = cProfile.Profile(); pr.enable(); analyze_workload(w); pr.disable()
    uninstall(prev)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
chk.close()
PY
