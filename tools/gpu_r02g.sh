mkdir -p gpurun_out
python - > gpurun_out/config3_strategies.jsonl 2>&1 <<'PY'
import json, os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from bench import entries, load_sites
from paper_2603_24595_b200.engine import SiteChecker, compile_all
chk = SiteChecker(device=0, compile_workers=0)
for probe in ("1", "0"):
    if probe == "0":
        os.environ["MK_NO_PROBE"] = "1"
    packed, _ = chk.pack([c for c, _ in compile_all(load_sites(entries('config3'))[1])])
    rs = chk.engine.upload(packed)
    runs = [rs.run({'max_seconds': 600.0}) for _ in range(5)]
    rs.free()
    print(json.dumps({"probe": probe, "device_ms": [round(r["device_ms"], 2) for r in runs],
                      "boxes": [r["boxes"] for r in runs], "strategy": [r["strategy"] for r in runs]}), flush=True)
PY
export MK_REAL_STRATEGY=0
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__thread_inst_executed.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_moe_align.csv python tools/profile_step.py moe_align > gpurun_out/step_moe_align.json 2> gpurun_out/step_moe_align.err
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_search -s 0 -c 3 -o gpurun_out/prof_moe_align -f python tools/profile_step.py moe_align > gpurun_out/ncu_full_moe_align.log 2>&1
