"""One oracle-rule access sweep (bench.py k2_access_replay: every recorded
access of fused_add_rms_norm at num_tokens T) between cudaProfilerStart/Stop
for ncu --profile-from-start off."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402
from refpath import add_reference, analyze_workload  # noqa: E402
from paper_2603_24595_b200 import replay  # noqa: E402
from paper_2603_24595_b200.detectors import install, uninstall  # noqa: E402
from paper_2603_24595_b200.engine import SiteChecker  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
FAST = len(sys.argv) > 2 and sys.argv[2] == "fast"   # owner-table path
assert add_reference()
torch.cuda.set_device(0)
chk = SiteChecker(device=0, compile_workers=0)
recs = []
prev = install(checker=chk, recorders=recs)
try:
    analyze_workload("fused_add_rms_norm")
finally:
    uninstall(prev)
records = [a for d in recs for a in d.accesses]
origin_of = recs[0].table.origin_of
launch = replay.launch_model(chk, records, origin_of, {"BS": 1, "SL": T})
accs, progs, key_bits, _ = replay.build(records, origin_of, launch)
grid = [launch[d] for d in replay.DIMS[:3]]
block = [launch[d] for d in replay.DIMS[3:]]
probs = [a.program.problem for a in accs]
nkeys = (1 << (key_bits - 1)) if FAST else 0
for _ in range(2):
    chk.engine.access_sweep(probs, progs, grid, block, key_bits, nkeys)
torch.cuda.synchronize()
torch.cuda.profiler.start()
r = chk.engine.access_sweep(probs, progs, grid, block, key_bits, nkeys)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(json.dumps(r))
chk.close()
