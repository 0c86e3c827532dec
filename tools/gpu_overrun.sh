# GPU box: where does a budgeted light config3 run spend time past its budget
mkdir -p gpurun_out
python - > gpurun_out/overrun.jsonl 2>&1 <<'PY'
import json, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from paper_2603_24595_b200.engine import SiteChecker, compile_all
qs = load_sites(entries("config3"))[1]
light = [c for c, _ in compile_all(qs, light=True) if c is not None]
for v in ["", "_A"]:
    chk = SiteChecker(device=0, compile_workers=0, lib_path=f"paper_2603_24595_b200/libmk_b200{v}.so")
    packed, _ = chk.pack(light)
    rs = chk.engine.upload(packed)
    for lim in ({"max_seconds": 0.5}, {"max_seconds": 0.5, "chunk": -2}, {"max_seconds": 0.1},
                {"max_seconds": 0.02}):
        for _ in range(2):
            r = rs.run(lim)
            print(json.dumps({"lib": v, "lim": lim, **{k: r[k] for k in ("device_ms", "seconds", "bb_ms", "leaf_ms", "rounds", "launches", "boxes", "points", "steps", "strategy")}}), flush=True)
    # per problem: run each unknown problem alone with 0.05 s and report the overrun
    import numpy as np
    st = rs.status[:len(packed.problems)].copy()
    rs.free()
    unk = [i for i, s in enumerate(st) if s == 2]
    worst = []
    for i in unk[:80]:
        r = chk.engine.solve([packed.problems[i]], {"max_seconds": 0.05})
        s = chk.engine.last_stats
        worst.append((round(s["device_ms"], 1), i, packed.problems[i].nvars, packed.problems[i].nregs, packed.problems[i].narrow))
    worst.sort(reverse=True)
    print(json.dumps({"lib": v, "single_problem_ms_top": worst[:15]}), flush=True)
    chk.close()
PY
