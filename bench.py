#!/usr/bin/env python
"""Checking-stage benchmark (one JSON line on rank 0).

A *step* decides every checker site query of one kernel x model
configuration (the queries the reference front end emits for it, recorded in
tests/golden/<workload>.json by oracle/gen_golden.py): verdict plus canonical
witness per site, i.e. the reference's Solver.check + canonicalize_witness
(engine/detectors.py, engine/report.py:147-203) for all sites at once.

metric  checked (thread, input) instances per second: the instances of all
        sites' compiled domains (thread identities x loop indices x havoc
        loads x user-controlled launch assignments, the boxes the engine
        certifies point by point or by interval proof) divided by the
        time-to-verdict of the step.  The same instance count is used by
        the reference arm, so the driver's ratio is the time-to-verdict
        ratio.
value   device-resident problem set (mk_set_eval), CUDA-event time on the
        engine stream; L2 flushed between steps.
e2e     the public API a user calls (SiteChecker.check_queries): compile,
        pack, H2D copy, search, D2H copy, witness assembly, every step.

--impl reference runs the reference's own checker (baseline/_ref, the
unmodified MiniKernel: Solver.check + canonicalize_witness) on the same
queries on the host cores; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_WORKLOAD = "rotary_embedding"   # BASELINE.json configs[1] (Llama-3-8B rotary)
CONFIG_NAMES = {
    "rms_norm": "vLLM rms_norm, Llama-2-7B (hidden 4096), num_tokens 1..2^20",
    "rotary_embedding": "vLLM rotary_embedding (NeoX), Llama-3-8B (32/8 heads, head 128), "
                        "symbolic positions and num_tokens 1..2^20",
    "moe_align": "fused-MoE moe_align_block_size port (Fig. 7), symbolic num_tokens x top_k",
    "fused_add_rms_norm": "vLLM fused_add_rms_norm (Fig. 2), hidden 7168, inferred context",
    "racy": "race probe (shared + global stores)",
    "paged_attention_v1": "vLLM paged_attention_v1, Mistral-7B (32/8 heads, head 128, block 16), "
                          "symbolic seq_len and block-table contents",
    "paged_attention_v2": "vLLM paged_attention_v2 (512-token partitions), Mistral-7B (32/8 heads, "
                          "head 128, block 16), symbolic seq_len and block-table contents",
    "moe_align_mixtral": "fused-MoE moe_align_block_size, Mixtral-8x7B (8 experts, top-2)",
    "topk_softmax": "fused-MoE topk_softmax, Mixtral-8x7B (8 experts, top-2)",
}


def _load_workload(name):
    from paper_2603_24595_b200 import ir
    from paper_2603_24595_b200.order import origin_lookup

    with open(os.path.join(ROOT, "tests", "golden", f"{name}.json")) as fh:
        doc = json.load(fh)
    queries = [([ir.from_json(a) for a in s["query"]], origin_lookup(s["origins"]))
               for s in doc["sites"]]
    return doc, queries


def _instances(compiled):
    """Instances certified per site: the volume of every compiled problem's
    root box (free symbols after exact presolve)."""
    per_site = []
    for cq, _ in compiled:
        v = 0
        if cq is not None:
            for p in cq.problems:
                v += p.volume()
        per_site.append(v)
    return per_site


class Clocks:
    """nvidia-smi samples during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int) -> None:
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def loop():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                         "--format=csv,noheader,nounits"],
                        capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()
        return self

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def _calibration(workload):
    """Per-unit calibration from the committed ncu capture of this workload
    (tools/gpu_profile.sh -> tools/summarize_ncu.py -> profiles/)."""
    path = os.path.join(ROOT, "profiles", f"ncu_{workload}_summary.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return {}


def _reference_checker_sample(queries, per_site, budget_s):
    """Reference's own checking stage (Solver.check + canonicalize_witness)
    on the site queries in order until ``budget_s`` of CPU time is spent."""
    from refbridge import reference_check_queries  # noqa: WPS433 (bench-local helper)

    t0 = time.perf_counter()
    done, inst = reference_check_queries(queries, budget_s=budget_s)
    dt = time.perf_counter() - t0
    return done, sum(per_site[:done]), dt


def _ref_job(name):
    """One reference job (kernel x model entry): every site query through the
    reference's Solver.check + canonicalize_witness; returns seconds."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from refbridge import reference_check_queries

    _, queries = _load_workload(name)
    t0 = time.perf_counter()
    done, _ = reference_check_queries(queries)
    assert done == len(queries)
    return time.perf_counter() - t0


def run_reference(args):
    """--impl reference: the unmodified reference checker on the host cores.
    At N ranks the arm checks the same N corpus entries as the B200 arm, one
    reference process per entry (the reference is single-threaded per job,
    SURVEY.md section 8d); only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from refbridge import have_reference

    if not have_reference():
        print(json.dumps({"impl": "reference",
                          "unavailable": "reference MiniKernel not installed under baseline/_ref"}))
        return
    from paper_2603_24595_b200.engine import compile_all

    if world > 1:
        names = ([args.workload] * world if args.workload != DEFAULT_WORKLOAD
                 else [CORPUS[i % len(CORPUS)] for i in range(world)])
    else:
        names = [args.workload]
    total = 0
    nsites = 0
    for n in names:
        _, queries = _load_workload(n)
        total += sum(_instances(compile_all(queries)))
        nsites += len(queries)
    cores = min(len(names), os.cpu_count() or 1)
    pool = None
    if len(names) > 1:
        import multiprocessing as mp

        pool = mp.get_context("fork").Pool(cores)
    times = []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if pool is None:
            _ref_job(names[0])
        else:
            pool.map(_ref_job, names)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    if pool is not None:
        pool.close()
    avg = sum(times) / len(times)
    value = total / avg
    out = {
        "impl": "reference",
        "metric": "checked (thread, input) access instances/sec; time-to-verdict per kernel x model",
        "value": value, "unit": "instances/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": avg * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int128 (mathematical integers)",
        "data": "recorded reference site queries", "time_to_verdict_ms": avg * 1e3,
        "config": {"workload": args.workload if world == 1 else "kernel x model corpus",
                   "description": CONFIG_NAMES.get(args.workload), "entries": names,
                   "sites": nsites},
        "cpu_baseline": {"value": value, "unit": "instances/s", "cores": cores,
                         "kind": "reference",
                         "sample": f"all {nsites} site queries of {len(names)} corpus entr"
                                   f"{'y' if len(names) == 1 else 'ies'} per step, reference "
                                   "Solver.check + canonicalize_witness, one process per entry"},
        "e2e": {"value": value, "unit": "instances/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


# BASELINE.json configs[4]: the kernel x model corpus of the rotary port,
# dealt one entry per rank under torchrun (weak scaling, no data-path
# collective); entry 0 is the N=1 headline workload (configs[1]).
CORPUS = ["rotary_embedding", "rotary_llama2_7b", "rotary_mistral_7b", "rotary_llama3_70b",
          "rotary_qwen2_7b", "rotary_llama2_13b", "rotary_mixtral_8x7b", "rotary_gemma_7b"]


def _analyze_line(chk, args, doc):
    """BASELINE metric part 2, time-to-verdict per kernel x model: the
    reference's own analyze() (parser, symbolic DFS, checking) on the
    workload's kernel port and context, once with the B200 checking stage and
    branch screening installed (GpuDetectors) and once unmodified; wall time
    of each and whether the findings are the reference's."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from refpath import add_reference, analyze_workload
    from goldens import expected_findings

    if not add_reference():
        return {"unavailable": "reference front end not installed under baseline/_ref"}
    from paper_2603_24595_b200.detectors import install, uninstall

    times = []
    for _ in range(3):
        prev = install(checker=chk, screening=True)
        t0 = time.perf_counter()
        try:
            got = analyze_workload(args.workload)
        finally:
            uninstall(prev)
        times.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    ref = analyze_workload(args.workload)
    ref_s = time.perf_counter() - t0
    return {"workload": args.workload, "b200_ms": 1e3 * min(times), "reference_ms": 1e3 * ref_s,
            "speedup": ref_s / min(times),
            "findings_equal_reference": got["findings"] == expected_findings(doc),
            "reference_findings_equal_golden": ref["findings"] == doc["findings"],
            "what": "analyze() wall time: reference front end (parser, DFS) + B200 checking "
                    "stage and branch screening vs the unmodified reference, one core"}


def _heavy_line(chk, args, int_peak, sm_mhz, sms):
    """The search kernels at scale: BASELINE configs[2] (paged attention,
    Mistral-7B), whose step is ~4e8 boxes, timed resident like the headline
    step; roofline from the same ncu calibration scheme."""
    doc, queries = _load_workload(args.heavy)
    from paper_2603_24595_b200.engine import compile_all

    compiled = compile_all(queries)
    packed, _ = chk.pack([c for c, _ in compiled])
    resident = chk.engine.upload(packed)
    lim = dict(chk.limits)
    lim["max_seconds"] = 600.0
    resident.run(lim)
    runs = [resident.run(lim) for _ in range(2)]
    resident.free()
    ms = sum(r["bb_ms"] + r["leaf_ms"] for r in runs) / len(runs)
    step_ms = sum(r["device_ms"] for r in runs) / len(runs)
    units = sum(r["boxes"] + r["points"] for r in runs) / len(runs)
    cal = _calibration(args.heavy)
    per_unit = cal.get("thread_inst_per_unit")
    achieved = units * per_unit / (ms / 1e3) if per_unit and ms > 0 else None
    return {"workload": args.heavy, "description": CONFIG_NAMES.get(args.heavy),
            "device_ms_per_step": step_ms, "boxes_and_instances_per_step": units,
            "roofline": {"bound": "int32-issue",
                         "achieved": achieved / 1e9 if achieved else None,
                         "peak": int_peak / 1e9, "unit": "Gop/s",
                         "frac": achieved / int_peak if achieved else None,
                         "kernel": "k_search (+k_bb, k_leaf)", "kernel_ms_per_step": ms,
                         "ops": f"SASS thread instructions per box/instance: {per_unit} (ncu, "
                                f"profiles/ncu_{args.heavy}_summary.json)",
                         "ncu_issue_active_pct": cal.get("k_search_issue_active_pct")}}


def _race_sweep_line(chk, args, peaks, src, int_peak):
    """K2 (race sweep, include/mk_b200.h mk_race_sweep) on config 1's output
    store (rms_norm, Llama-2-7B hidden 4096: out[blockIdx.x * hidden + idx])
    replayed at a full concrete launch: every (thread, loop iteration) access
    of the launch is evaluated and checked for conflicts.

    The sweep that runs is the fused ordered pass (the store is coalesced, so
    its keys arrive in order and the stable sort is the identity): one
    NVRTC-specialised kernel, no tuples in HBM, integer-issue bound; its
    roofline is thread instructions per instance (ncu, profiles/
    ncu_k2_summary.json) x instances / kernel time over 148 SMs x 128 lanes x
    clock.  ``sort_path`` runs the same tuples through the HBM radix-sort path
    (MK_RACE_FORCE_SORT): algorithmic bytes = 4 x tuple bytes per access
     / device time, against the HBM peak."""
    from paper_2603_24595_b200 import race

    doc, queries = _load_workload("rms_norm")
    T = args.race_tokens
    launch = {"BS": 1, "SL": T, "TC": T, "blockDim.x": 1024, "blockDim.y": 1, "blockDim.z": 1,
              "gridDim.x": T, "gridDim.y": 1, "gridDim.z": 1}
    progs = [race.race_program(a, o, launch) for s, (a, o) in zip(doc["sites"], queries)
             if s["site"] == "store_site" and s["line"] == 20]
    prog = max(progs, key=lambda p: p.instances)

    def timed(env):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            for _ in range(2):
                chk.engine.race_sweep(prog)
            return [chk.engine.race_sweep(prog) for _ in range(3)]
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v

    runs = timed({})
    ms = sum(r["gen_ms"] + r["sort_ms"] + r["scan_ms"] for r in runs) / len(runs)
    r = runs[-1]
    cal = _calibration("k2")
    per_inst = cal.get("thread_inst_per_instance")
    kms = sum(x["gen_ms"] for x in runs) / len(runs)
    achieved = prog.instances * per_inst / (kms / 1e3) / 1e9 if per_inst and kms > 0 else None
    sruns = timed({"MK_RACE_FORCE_SORT": "1"})
    sms_ = sum(x["gen_ms"] + x["sort_ms"] + x["scan_ms"] for x in sruns) / len(sruns)
    sr = sruns[-1]
    hbm_peak = peaks.get("hbm_gbs", 6650.0) if isinstance(peaks, dict) else 6650.0
    s_ach = sr["hbm_bytes"] / (sms_ / 1e3) / 1e9
    return {"workload": f"rms_norm output store (BASELINE configs[0]) at num_tokens={T}: "
                        f"{T} blocks x 1023 threads x 4 iterations",
            "accesses": r["tuples"], "instances": prog.instances, "has_race": bool(r["has_race"]),
            "path": "fused ordered pass" if r["fused"] else ("in-order scan" if r["sorted"] else "radix sort"),
            "ms": ms, "instances_per_s": prog.instances / (ms / 1e3),
            "gen_ms": r["gen_ms"], "sort_ms": r["sort_ms"], "scan_ms": r["scan_ms"],
            "roofline": {"bound": "int32-issue",
                         "achieved": achieved, "peak": int_peak / 1e9, "unit": "Gop/s",
                         "frac": achieved * 1e9 / int_peak if achieved else None,
                         "traffic": r["hbm_bytes"],
                         "kernel": "mk_race_fused_jit (NVRTC, sm_100a)",
                         "ops": f"SASS thread instructions per instance: {per_inst} "
                                "(ncu, profiles/ncu_k2_summary.json)"},
            "sort_path": {"ms": sms_, "gen_ms": sr["gen_ms"], "sort_ms": sr["sort_ms"],
                          "scan_ms": sr["scan_ms"], "sort_key_bits": sr["sort_bits"],
                          "same_result": (sr["tuples"], sr["conflicts"], sr["has_race"]) ==
                                         (r["tuples"], r["conflicts"], r["has_race"]),
                          "roofline": {"bound": "hbm", "achieved": s_ach, "peak": hbm_peak,
                                       "unit": "GB/s", "frac": s_ach / hbm_peak, "traffic": None,
                                       "algorithmic_bytes": sr["hbm_bytes"],
                                       "peak_source": f"peaks file: {src}"}}}


def _race_sharded_line(chk, args, world):
    """K2 across the ranks (shard.race_sweep_sharded): config 1's output
    store at the N=1 line's launch (num_tokens = --race-tokens; strong
    scaling: a launch's instance indices are 32-bit, < 2^31), each rank a
    contiguous instance range through the fused pass, one all_gather_object
    of the shard summaries.  Time: max over ranks of the call (device pass +
    combine)."""
    import torch
    import torch.distributed as dist

    from paper_2603_24595_b200 import race, shard

    doc, queries = _load_workload("rms_norm")
    T = args.race_tokens
    launch = {"BS": 1, "SL": T, "TC": T, "blockDim.x": 1024, "blockDim.y": 1, "blockDim.z": 1,
              "gridDim.x": T, "gridDim.y": 1, "gridDim.z": 1}
    progs = [race.race_program(a, o, launch)
             for s, (a, o) in zip(doc["sites"], queries)
             if s["site"] == "store_site" and s["line"] == 20]
    prog = max(progs, key=lambda p: p.instances)
    for _ in range(2):
        shard.race_sweep_sharded(chk.engine, prog)
    times = []
    for _ in range(3):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        got = shard.race_sweep_sharded(chk.engine, prog)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    t = torch.tensor([min(times)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) * 1e3
    return {"workload": f"rms_norm output store at num_tokens={T} ({world} shards)",
            "instances": prog.instances, "accesses": got["tuples"], "has_race": bool(got["has_race"]),
            "ms": ms, "instances_per_s": prog.instances / (ms / 1e3), "scaling": "strong",
            "what": "max over ranks of race_sweep_sharded (fused pass on the rank's range + "
                    "all_gather_object of the shard summaries), wall clock around synchronized calls"}


def _access_line(chk, args, peaks, src, int_peak):
    """K2 with the specification's oracle rule (paper_2603_24595_b200.replay,
    mk_access_sweep): every load and store the reference front end executes
    on fused_add_rms_norm (Fig. 2, hidden 7168; in-place residual update,
    shared reduction with a barrier) replayed at num_tokens = --access-tokens:
    granule tuples of all accesses to written regions, radix-sorted in HBM,
    segmented read-write / write-write scan.  The path that runs on a
    race-free launch is the owner-table pass (integer-issue roofline, ncu
    calibration profiles/ncu_access_summary.json); ``sort_path`` times the
    radix-sort path on the same accesses, HBM roofline: algorithmic bytes =
    4 x 16 B per tuple (8 B key + 8 B value; one write at
    generation, one read + one write for a single-pass-equivalent sort, one
    read in the scan) / device time."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from refpath import add_reference, analyze_workload

    if not add_reference():
        return {"unavailable": "reference front end not installed under baseline/_ref"}
    from paper_2603_24595_b200 import replay
    from paper_2603_24595_b200.detectors import install, uninstall

    name = "fused_add_rms_norm"
    recs = []
    prev = install(checker=chk, recorders=recs)
    try:
        analyze_workload(name)
    finally:
        uninstall(prev)
    records = [a for d in recs for a in d.accesses]
    origin_of = recs[0].table.origin_of
    T = args.access_tokens
    launch = replay.launch_model(chk, records, origin_of, {"BS": 1, "SL": T})
    for _ in range(2):
        replay.replay_races(chk.engine, records, origin_of, launch)
    runs = []
    for _ in range(3):
        t0 = time.perf_counter()
        r = replay.replay_races(chk.engine, records, origin_of, launch)
        runs.append((time.perf_counter() - t0, r))
    res = runs[-1][1]
    # device phases of the last call (the result carries no timings: take them
    # from one direct sweep of the same layout)
    accs, progs, key_bits, _ = replay.build(records, origin_of, launch)
    grid = [launch[d] for d in replay.DIMS[:3]]
    block = [launch[d] for d in replay.DIMS[3:]]
    probs = [a.program.problem for a in accs]
    dev = [chk.engine.access_sweep(probs, progs, grid, block, key_bits, nkeys=1 << (key_bits - 1))
           for _ in range(3)]
    old = os.environ.get("MK_ACCESS_NO_FAST")
    os.environ["MK_ACCESS_NO_FAST"] = "1"
    try:
        srt = [chk.engine.access_sweep(probs, progs, grid, block, key_bits) for _ in range(3)]
    finally:
        if old is None:
            os.environ.pop("MK_ACCESS_NO_FAST", None)
    sort_ms = sum(d["gen_ms"] + d["sort_ms"] + d["scan_ms"] for d in srt) / len(srt)
    ms = sum(d["gen_ms"] + d["sort_ms"] + d["scan_ms"] for d in dev) / len(dev)
    hbm_peak = peaks.get("hbm_gbs", 6650.0) if isinstance(peaks, dict) else 6650.0
    algo = 4 * 16 * res.tuples
    s_ach = algo / (sort_ms / 1e3) / 1e9
    # owner-table pass: integer-issue bound (no tuples in HBM); thread
    # instructions per instance from the committed ncu launch list
    cal = _calibration("access")
    per_inst = cal.get("thread_inst_per_instance")
    ach = res.instances * per_inst / (ms / 1e3) / 1e9 if per_inst and ms > 0 else None
    return {"workload": f"{name} (Fig. 2, hidden 7168) at num_tokens={T}, launch "
                        f"<<<{grid[0]}; {block[0]}>>>: every recorded access of a written region",
            "accesses": res.accesses, "instances": res.instances, "tuples": res.tuples,
            "has_race": res.has_race, "racy_granules": res.racy, "key_bits": key_bits,
            "device_ms": ms, "gen_ms": dev[-1]["gen_ms"], "sort_ms": dev[-1]["sort_ms"],
            "scan_ms": dev[-1]["scan_ms"], "wall_ms": 1e3 * min(t for t, _ in runs),
            "tuples_per_s": res.tuples / (ms / 1e3),
            "path": "owner table (race-free, no sort)" if dev[-1]["fast"] else "radix sort",
            "roofline": {"bound": "int32-issue", "achieved": ach, "peak": int_peak / 1e9,
                         "unit": "Gop/s", "frac": ach * 1e9 / int_peak if ach else None,
                         "traffic": cal.get("dram_bytes"),
                         "kernel": "mk_access_jit (NVRTC, sm_100a), owner-table write + read passes",
                         "ops": f"SASS thread instructions per instance: {per_inst} "
                                "(ncu, profiles/ncu_access_summary.json)"},
            "sort_path": {"ms": sort_ms, "gen_ms": srt[-1]["gen_ms"], "sort_ms": srt[-1]["sort_ms"],
                          "scan_ms": srt[-1]["scan_ms"],
                          "same_result": (srt[-1]["has_race"], srt[-1]["tuples"]) ==
                                         (dev[-1]["has_race"], dev[-1]["tuples"]),
                          "roofline": {"bound": "hbm", "achieved": s_ach, "peak": hbm_peak,
                                       "unit": "GB/s", "frac": s_ach / hbm_peak, "traffic": None,
                                       "algorithmic_bytes": algo}}}


def run_b200(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: MK_BENCH_ONE_DEVICE runs every rank on cuda:0 over gloo, so
    # the N>1 path can be exercised on a one-GPU box (never for numbers)
    one = bool(os.environ.get("MK_BENCH_ONE_DEVICE"))
    if one:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2603_24595_b200 import shard
    from paper_2603_24595_b200.engine import SiteChecker, compile_all

    if world > 1:
        if args.workload != DEFAULT_WORKLOAD:
            names = [args.workload] * world
        else:
            names = [CORPUS[i % len(CORPUS)] for i in range(world)]
    else:
        names = [args.workload]
    my_name = names[rank]
    doc, queries = _load_workload(my_name)
    compiled = compile_all(queries)
    per_site = _instances(compiled)
    instances = sum(per_site)
    chk = SiteChecker(device=local)
    packed, offsets = chk.pack([c for c, _ in compiled])
    resident = chk.engine.upload(packed)
    limits = dict(chk.limits)
    limits["max_seconds"] = min(chk.limits["max_seconds"] * len(queries), 3600.0)

    # parity gate: the benchmarked result must be the reference's (sites the
    # reference only timed out on are pinned by its own z3 path, see
    # tests/goldens.py and oracle/z3_crosscheck.py)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from goldens import mismatches

    results = chk.decide(compiled, packed, offsets)
    bad = mismatches(doc, results)
    if bad:
        raise SystemExit(f"parity failure on {my_name} sites {bad[:10]}")

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    for _ in range(args.warmup):
        resident.run(limits)
    clocks = Clocks(local).start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    dev_ms, wall, launches = [], [], 0
    stats_acc = {}
    for _ in range(args.steps):
        flush.random_(0, 255)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = resident.run(limits)
        wall.append(time.perf_counter() - t0)
        dev_ms.append(st["device_ms"])
        launches += int(st["launches"])
        for k, v in st.items():
            stats_acc[k] = stats_acc.get(k, 0) + v
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms_step = sum(dev_ms) / len(dev_ms)
    total_instances = float(instances)
    if world > 1:
        t = torch.tensor([ms_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
        t = torch.tensor([float(instances)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        total_instances = float(t.item())
    value = total_instances / (ms_step / 1e3)

    # e2e through the public API with host buffers (compile + H2D + search +
    # D2H + witness assembly); at N>1 the corpus call deals one entry per rank
    # and all-gathers every result to every rank.  Warm-up calls start the
    # host compile workers outside the timed steps.
    entries = None
    if world > 1:
        entries = [_load_workload(n)[1] for n in names]

    def e2e_call():
        if entries is None:
            return chk.check_queries(queries)
        return shard.check_corpus(chk, entries)

    for _ in range(args.warmup):
        e2e_call()
    e2e_t = []
    for step in range(max(1, args.steps)):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        res = e2e_call()
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = sum(e2e_t) / len(e2e_t)
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    # roofline of the dominant kernels (pre-split + persistent search; one
    # box / instance = one unit): integer-lane issue.  Achieved = units per
    # step (live engine counters) x SASS thread instructions per unit (ncu
    # capture of the same workload, profiles/ncu_<workload>_summary.json)
    # / device time of those kernels (CUDA events on the engine streams).
    n = args.steps
    search_ms = stats_acc["bb_ms"] / n + stats_acc["leaf_ms"] / n
    units = (stats_acc["boxes"] + stats_acc["points"]) / n
    insns = (stats_acc["insns_bb"] + stats_acc["insns_leaf"]) / n
    peaks, src = _peaks()
    sm_mhz = clk["sm_mhz"] or peaks.get("sm_max_mhz", 1965.0)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    int_peak = sms * 128 * sm_mhz * 1e6           # 128 INT32 lanes / SM / clock (B200: 148 SMs)
    cal = _calibration(args.workload)
    per_unit = cal.get("thread_inst_per_unit")
    if per_unit:
        achieved = units * per_unit / (search_ms / 1e3) if search_ms > 0 else 0.0
        ops = (f"SASS thread instructions: {units:.3g} boxes+instances per step x "
               f"{per_unit:.1f} per unit (ncu, profiles/ncu_{args.workload}_summary.json)")
    else:
        achieved = insns / (search_ms / 1e3) if search_ms > 0 else 0.0
        ops = "bytecode instructions executed (no ncu calibration committed)"

    k2 = _race_sweep_line(chk, args, peaks, src, int_peak) if rank == 0 and args.race_tokens > 0 else None
    k2_sharded = (_race_sharded_line(chk, args, world)
                  if world > 1 and args.race_tokens > 0 else None)
    analyze = _analyze_line(chk, args, doc) if rank == 0 and world == 1 and args.analyze else None
    access = (_access_line(chk, args, peaks, src, int_peak)
              if rank == 0 and world == 1 and args.access_tokens > 0 else None)
    heavy = (_heavy_line(chk, args, int_peak, sm_mhz, sms)
             if rank == 0 and world == 1 and args.heavy and args.heavy != args.workload else None)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        try:
            from refbridge import have_reference, reference_check_queries
            if have_reference():
                t0 = time.perf_counter()
                done, _ = reference_check_queries(queries, budget_s=args.cpu_budget)
                dt = time.perf_counter() - t0
                cpu = {"value": sum(per_site[:done]) / dt, "unit": "instances/s", "cores": 1,
                       "kind": "reference",
                       "sample": f"first {done} of {len(queries)} {args.workload} site queries "
                                 "through the reference's Solver.check + canonicalize_witness "
                                 f"(baseline/_ref), {dt:.1f}s, 1 thread"}
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "instances/s", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        out = {
            "metric": "checked (thread, input) access instances/sec; time-to-verdict per kernel x model",
            "value": value, "unit": "instances/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int128 (mathematical integers)",
            "data": "site queries recorded from the reference front end on the workload port",
            "config": {"workload": args.workload if world == 1 else "kernel x model corpus",
                       "description": CONFIG_NAMES.get(args.workload) if world == 1 else
                       "rotary_embedding port under one model context per rank",
                       "entries": names,
                       "sites": len(queries), "instances_per_step": total_instances,
                       "l2": "flushed between steps (256 MiB write)",
                       "parallelism": "1 GPU" if world == 1 else
                       f"{world} ranks, one corpus entry each (no data-path collective; "
                       "results all-gathered in e2e)"},
            "time_to_verdict_ms": ms_step,
            "wall_ms_per_step": 1e3 * sum(wall) / len(wall),
            "evaluated_per_step": {"boxes": stats_acc["boxes"] / n, "points": stats_acc["points"] / n},
            "e2e": {"value": total_instances / e2e_s, "unit": "instances/s",
                    "h2d_bytes_per_step": packed.host_bytes(),
                    "d2h_bytes_per_step": resident.d2h_bytes(), "ms_per_step": e2e_s * 1e3},
            "roofline": {"bound": "int32-issue", "achieved": achieved / 1e9,
                         "peak": int_peak / 1e9, "unit": "Gop/s",
                         "frac": achieved / int_peak if int_peak else None,
                         "traffic": cal.get("k_search_dram_bytes_per_launch"),
                         "kernel": "k_search (+k_bb pre-split, k_leaf)",
                         "kernel_ms_per_step": search_ms,
                         "units_per_step": units,
                         "bytecode_insns_per_step": insns,
                         "ops": ops,
                         "ncu_issue_active_pct": cal.get("k_search_issue_active_pct"),
                         "peak_source": f"{sms} SMs x 128 INT32 lanes x {sm_mhz:.0f} MHz "
                                        f"(clock sampled; peaks file: {src})"},
            "cpu_baseline": cpu,
            "k2_race_sweep": k2,
            "k2_access_replay": access,
            "k2_race_sharded": k2_sharded,
            "time_to_verdict": analyze,
            "k1_heavy": heavy,
            "clocks": clk,
            "gpu_launches": launches,
        }
        print(json.dumps(out))
    resident.free()
    chk.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-analyze", dest="analyze", action="store_false",
                    help="skip the end-to-end analyze() time-to-verdict line")
    ap.add_argument("--heavy", default="paged_attention_v1",
                    help="workload of the k1_heavy line ('' to skip)")
    ap.add_argument("--access-tokens", type=int, default=16384,
                    help="num_tokens of the oracle-rule access replay line (0: skip)")
    ap.add_argument("--race-tokens", type=int, default=262144,
                    help="num_tokens of the K2 race-sweep line (0: skip)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
