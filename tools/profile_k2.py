"""One K2 race sweep (config 1's output store at a full concrete launch)
between cudaProfilerStart/Stop, for ncu --profile-from-start off: the launch
list gives each sweep kernel's time and DRAM bytes."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402
from goldens import load, queries  # noqa: E402
from paper_2603_24595_b200 import race  # noqa: E402
from paper_2603_24595_b200.engine import SiteChecker  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
torch.cuda.set_device(0)
chk = SiteChecker(device=0, compile_workers=0)
doc = load("rms_norm")
qs = queries(doc)
launch = {"BS": 1, "SL": T, "TC": T, "blockDim.x": 1024, "blockDim.y": 1, "blockDim.z": 1,
          "gridDim.x": T, "gridDim.y": 1, "gridDim.z": 1}
progs = [race.race_program(a, o, launch) for s, (a, o) in zip(doc["sites"], qs)
         if s["site"] == "store_site" and s["line"] == 20]
prog = max(progs, key=lambda p: p.instances)
for _ in range(2):
    chk.engine.race_sweep(prog)
torch.cuda.synchronize()
torch.cuda.profiler.start()
r = chk.engine.race_sweep(prog)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
r.pop("pair", None)
print(json.dumps(r))
chk.close()
