"""Development aid: K2 race sweep of config 1's output store (rms_norm,
Llama-2-7B hidden 4096) at a concrete num_tokens."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from goldens import load, queries  # noqa: E402
from paper_2603_24595_b200 import race  # noqa: E402
from paper_2603_24595_b200.native import Engine  # noqa: E402

eng = Engine(0)
doc = load("rms_norm")
for T in [int(x) for x in sys.argv[1:]] or [4096, 65536, 131072]:
    launch = {"BS": 1, "SL": T, "TC": T, "blockDim.x": 1024, "blockDim.y": 1, "blockDim.z": 1,
              "gridDim.x": T, "gridDim.y": 1, "gridDim.z": 1}
    for s, (a, o) in zip(doc["sites"], queries(doc)):
        if s["site"] == "store_site" and s["line"] == 20:
            prog = race.race_program(a, o, launch)
            if prog.instances < 1 << 20:
                continue
            for rep in range(3):
                t0 = time.perf_counter()
                got = eng.race_sweep(prog)
                wall = time.perf_counter() - t0
            ms = got["gen_ms"] + got["sort_ms"] + got["scan_ms"]
            got.pop("pair", None)
            print(json.dumps({"T": T, "jit_env": os.environ.get("MK_NO_JIT"), "instances": prog.instances, "wall_ms": wall * 1e3,
                              "device_ms": ms, "algo_GBps": got["hbm_bytes"] / ms / 1e6, **got}),
                  flush=True)
