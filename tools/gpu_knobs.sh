# GPU box: resident full-presolve step device time per search knob setting
# (MK_SPLIT_K split arity, MK_ADAPT_K shallow-stack widening, MK_TASK_GROUP
# tasks per grab), read by the engine at every call.  KNOBS="NAME=v1,v2 ..."
# picks the settings swept (default: split arity x widening)
mkdir -p gpurun_out
python - > gpurun_out/knobs.jsonl 2>&1 <<'PY'
import json, os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from paper_2603_24595_b200.engine import SiteChecker, compile_all
chk = SiteChecker(device=0, compile_workers=0)
sets = {}
for g in ["config3", "moe_align", "paged_attention_v2_long_b16", "paged_attention_v1", "racy"]:
    packed, _ = chk.pack([c for c, _ in compile_all(load_sites(entries(g))[1]) if c is not None])
    sets[g] = chk.engine.upload(packed)
import itertools
spec = os.environ.get("KNOBS", "MK_SPLIT_K=6,8,12,16 MK_ADAPT_K=0,1").split()
names = [x.split("=")[0] for x in spec]
for vals in itertools.product(*[x.split("=")[1].split(",") for x in spec]):
    for n, v in zip(names, vals):
        os.environ[n] = v
    for g, rs in sets.items():
        runs = [rs.run({"max_seconds": 600.0}) for _ in range(5)]
        print(json.dumps({**dict(zip(names, vals)), "group": g,
                          "ms": sorted(round(r["device_ms"], 2) for r in runs),
                          "boxes": runs[-1]["boxes"], "steps": runs[-1]["steps"]}), flush=True)
PY
