"""Summarise the ncu launch list of one K2 sweep (tools/profile_k2.py under
ncu --metrics gpu__time_duration.sum,smsp__thread_inst_executed.sum,...)
into profiles/ncu_k2_summary.json: per-kernel time, DRAM bytes and SASS
thread instructions, and thread instructions per instance of the fused pass
(bench.py's K2 roofline calibration)."""
import csv
import json
import sys

launches, step, out = sys.argv[1], sys.argv[2], sys.argv[3]
kernel = sys.argv[4] if len(sys.argv) > 4 else "mk_race_fused_jit"
st = json.loads(open(step).read().strip().splitlines()[-1])
rows = list(csv.reader(open(launches)))
hdr = None
per = {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", ""))
        per.setdefault(k, {}).setdefault(d["Metric Name"], 0.0)
        per[k][d["Metric Name"]] += v
res = {"source": "tools/profile_k2.py (rms_norm output store, num_tokens 262144)"
       if kernel == "mk_race_fused_jit" else
       "tools/profile_access.py (fused_add_rms_norm accesses, num_tokens 16384)",
       "instances": st["instances"], "accesses": st["tuples"], "kernels": per}
f = per.get(kernel)
if f and f.get("smsp__thread_inst_executed.sum"):
    res["thread_inst_per_instance"] = f["smsp__thread_inst_executed.sum"] / st["instances"]
    res["warp_inst_per_instance"] = f.get("smsp__inst_executed.sum", 0.0) / st["instances"]
    res["kernel_us"] = f.get("gpu__time_duration.sum", 0.0) / 1e3
    res["dram_bytes"] = f.get("dram__bytes_read.sum", 0.0) + f.get("dram__bytes_write.sum", 0.0)
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
