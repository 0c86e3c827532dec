"""Summarise an ncu launch list + full capture into profiles/ (round-tagged)."""
import csv, io, json, os, subprocess, sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        name = name.split("(")[0].split("<")[0].strip()
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
        per[name][0] += 1
        per[name][1] += v * scale
    tot = sum(v[1] for v in per.values()) or 1.0
    return {k: {"launches": v[0], "total_us": round(v[1], 1), "share": round(v[1] / tot, 4)}
            for k, v in sorted(per.items(), key=lambda kv: -kv[1][1])}


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed.sum.per_cycle_elapsed", "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active",
            "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sass__inst_executed_local_loads", "sass__inst_executed_local_stores",
            "sm__cycles_elapsed.avg"]
    res = {}
    for i, h in enumerate(hdr):
        if h in want:
            res[h] = f"{vals[i]} {units[i]}".strip()
    return res


def main(workload, tag):
    g = os.path.join(ROOT, "gpurun_out")
    summ = {"workload": workload, "round": tag}
    lp = os.path.join(g, f"launches_{workload}.csv")
    if os.path.exists(lp):
        summ["launch_list"] = launches(lp)
    rp = os.path.join(g, f"prof_{workload}.ncu-rep")
    if os.path.exists(rp):
        summ["k_search_full"] = full(rp)
        f = summ["k_search_full"]
        def num(k, scale):
            v = f.get(k, "0 x").split()
            x = float(v[0].replace(",", ""))
            u = v[1] if len(v) > 1 else ""
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        summ["k_search_dram_bytes_per_launch"] = num("dram__bytes_read.sum", 1) + num("dram__bytes_write.sum", 1)
    bp = os.path.join(g, f"bench_{workload}.json")
    if os.path.exists(bp):
        summ["bench_line"] = json.loads(open(bp).read().strip().splitlines()[-1])
    rp2 = os.path.join(g, f"bench_ref_{workload}.json")
    if os.path.exists(rp2):
        summ["reference_line"] = json.loads(open(rp2).read().strip().splitlines()[-1])
    out = os.path.join(ROOT, "profiles", f"{tag}_{workload}.json")
    json.dump(summ, open(out, "w"), indent=1)
    json.dump({"k_search_dram_bytes_per_launch": summ.get("k_search_dram_bytes_per_launch")},
              open(os.path.join(ROOT, "profiles", f"ncu_{workload}_summary.json"), "w"))
    print(json.dumps({k: v for k, v in summ.items() if k != "bench_line" and k != "reference_line"}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "r01")
