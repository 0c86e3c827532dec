"""Summarise one tools/gpu_profile.sh session into profiles/ (round-tagged).

Inputs (gpurun_out/): launches_<W>.csv (ncu launch list of one resident step:
per-launch duration, thread- and warp-level instructions), step_<W>.json (the
engine statistics of that step), prof_<W>.ncu-rep (ncu --set full of the
persistent search kernel), bench_<W>.json / bench_ref_<W>.json.

Outputs: profiles/<tag>_<W>.json (everything) and
profiles/ncu_<W>_summary.json (the per-unit calibration bench.py reads:
SASS thread instructions the engine kernels issue per box / instance, and
DRAM bytes per search launch)."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ENGINE_KERNELS = ("k_search", "k_bb", "k_leaf")


def _short(name):
    name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    if name.startswith("void "):
        name = name[5:]
    return name.split("(")[0].strip()


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(lambda: defaultdict(float))
    count = defaultdict(set)
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = _short(d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", ""))
        m = d.get("Metric Name")
        if m == "gpu__time_duration.sum":
            unit = d.get("Metric Unit", "ns")
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                  "msecond": 1e3}.get(unit, 1e-3)
            m = "time_us"
        per[name][m] += v
        count[name].add(d["ID"])
    tot = sum(v.get("time_us", 0.0) for v in per.values()) or 1.0
    out = {}
    for k, v in sorted(per.items(), key=lambda kv: -kv[1].get("time_us", 0.0)):
        out[k] = {"launches": len(count[k]), "total_us": round(v.get("time_us", 0.0), 1),
                  "share": round(v.get("time_us", 0.0) / tot, 4),
                  "thread_inst": v.get("smsp__thread_inst_executed.sum", 0.0),
                  "warp_inst": v.get("smsp__inst_executed.sum", 0.0)}
    return out


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    # the longest captured launch (the steady-state search, not the dive)
    it = hdr.index("gpu__time_duration.sum")
    vals = max(rows[2:], key=lambda r: float(r[it].replace(",", "") or 0))
    want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed.sum.per_cycle_elapsed",
            "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active",
            "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "sass__inst_executed_local_loads",
            "sass__inst_executed_local_stores", "sm__cycles_elapsed.avg",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"]
    res = {}
    for i, h in enumerate(hdr):
        if h in want:
            res[h] = f"{vals[i]} {units[i]}".strip()
    return res


def _bytes(s):
    v = s.split()
    x = float(v[0].replace(",", ""))
    u = v[1] if len(v) > 1 else ""
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main(workload, tag):
    g = os.path.join(ROOT, "gpurun_out")
    summ = {"workload": workload, "round": tag}
    calib = {"workload": workload, "round": tag}
    lp = os.path.join(g, f"launches_{workload}.csv")
    sp = os.path.join(g, f"step_{workload}.json")
    if os.path.exists(lp):
        summ["launch_list"] = launches(lp)
    if os.path.exists(sp):
        summ["step_stats"] = json.loads(open(sp).read().strip().splitlines()[-1])["stats"]
    if "launch_list" in summ and "step_stats" in summ:
        ll, st = summ["launch_list"], summ["step_stats"]
        eng = {k: v for k, v in ll.items() if k.startswith(ENGINE_KERNELS)}
        units = st["boxes"] + st["points"]
        ti = sum(v["thread_inst"] for v in eng.values())
        calib["thread_inst_per_unit"] = ti / units if units else None
        calib["units_per_step"] = units
        calib["engine_kernel_us"] = sum(v["total_us"] for v in eng.values())
        calib["engine_share_of_step"] = sum(v["share"] for v in eng.values())
    rp = os.path.join(g, f"prof_{workload}.ncu-rep")
    if os.path.exists(rp):
        summ["k_search_full"] = f = full(rp)
        calib["k_search_dram_bytes_per_launch"] = (_bytes(f.get("dram__bytes_read.sum", "0"))
                                                   + _bytes(f.get("dram__bytes_write.sum", "0")))
        calib["k_search_issue_active_pct"] = f.get(
            "smsp__issue_active.avg.pct_of_peak_sustained_active")
    bp = os.path.join(g, f"bench_{workload}.json")
    if os.path.exists(bp) and os.path.getsize(bp):
        summ["bench_line"] = json.loads(open(bp).read().strip().splitlines()[-1])
    rp2 = os.path.join(g, f"bench_ref_{workload}.json")
    if os.path.exists(rp2) and os.path.getsize(rp2):
        summ["reference_line"] = json.loads(open(rp2).read().strip().splitlines()[-1])
    summ["calibration"] = calib
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    json.dump(summ, open(os.path.join(ROOT, "profiles", f"{tag}_{workload}.json"), "w"),
              indent=1)
    json.dump(calib, open(os.path.join(ROOT, "profiles", f"ncu_{workload}_summary.json"), "w"),
              indent=1)
    print(json.dumps({k: v for k, v in summ.items()
                      if k not in ("bench_line", "reference_line")}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "r01")
