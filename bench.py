#!/usr/bin/env python
"""Checking-stage benchmark (one JSON line on rank 0).

A *step* decides every checker site query of one workload: verdict plus
canonical witness per site, i.e. the reference's Solver.check +
canonicalize_witness (engine/detectors.py:97-298, engine/report.py:147-203)
for all sites at once.  The queries are the ones the reference front end
emits on the workload's kernel ports (recorded in tests/golden/ by
oracle/gen_golden.py).

Default workload: BASELINE.json configs[2] at its stated domain (SURVEY.md
8(d)): vLLM paged_attention v1 with block sizes 8 / 16 / 32 and v2
(512-token partitions), Mistral-7B, seq_len up to 2^20, a 2^20-block KV cache
(workloads/paged_attention_*_long_*).  ``--workload corpus`` is configs[4]
(every golden workload); any single workload name works too.

Instances.  A site's instances are the points of its domain after
structural lowering (thread identities x loop indices x havoc loads x
user-controlled launch assignments): the root-box volumes of its light
compile's device problems (its full compile's when the light one cannot
bound it; bench.site_instances).  Both arms use the same per-site counts,
so every ratio of values is a ratio of times.

Two tiers (SiteChecker.check_queries): every site is first compiled light
(structural presolve only) and searched on the device within a short
budget; the sites the device does not decide there go through the full
host presolve and the device.  ``decided`` reports where each verdict came
from.

value   instances / device time of the step: both tiers' problem sets
        resident in HBM (mk_set_eval), CUDA events on the engine streams, L2
        flushed between steps (256 MiB write).  Max over ranks.
e2e     the same instances / wall time of the public API a user calls
        (SiteChecker.check_queries; N>1: shard.check_sites): host compile on
        the worker pool, pack, H2D, search, D2H, witness assembly, every step.
roofline  integer issue of the dominant kernel k_search against the INT32
        issue peak measured on this device (mk_int_peak): algorithmic basis =
        bytecode instructions evaluated (live device counters, SURVEY.md
        8(d)); the SASS-issue basis (ncu calibration) is reported beside it.

--gpus N without torchrun re-launches itself under torch.distributed.run;
the sites are dealt across the ranks (strong scaling, no data-path
collective; one all_gather_object of the verdict records in e2e).

--impl reference runs the reference's own checker (baseline/_ref, the
unmodified MiniKernel: Solver.check + canonicalize_witness) on the same site
queries on the host cores, rank 0 only: each step decides the next slice of
the site list on a process pool (the reference is single-threaded per
query), so the K timed steps together decide every site once.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))

DEFAULT_WORKLOAD = "config3"
GROUPS = {
    "config3": ["paged_attention_v1_long_b8", "paged_attention_v1_long_b16",
                "paged_attention_v1_long_b32", "paged_attention_v2_long_b16"],
}
CONFIG_NAMES = {
    "config3": "BASELINE configs[2] at its stated domain: vLLM paged_attention v1 (block 8, 16, 32) "
               "and v2 (block 16, 512-token partitions, max_num_seqs 1024), Mistral-7B (32/8 heads, "
               "head 128), symbolic seq_len <= 2^20, block-table contents in [0, 2^20)",
    "corpus": "BASELINE configs[4]: every registered kernel x model workload (tests/golden)",
    "rms_norm": "vLLM rms_norm, Llama-2-7B (hidden 4096), num_tokens 1..2^20",
    "rotary_embedding": "vLLM rotary_embedding (NeoX), Llama-3-8B, symbolic positions and "
                        "num_tokens 1..2^20",
    "moe_align": "fused-MoE moe_align_block_size port (Fig. 7), symbolic num_tokens x top_k",
    "paged_attention_v1": "vLLM paged_attention_v1, Mistral-7B, block 16, seq_len <= 32768",
}


def entries(workload):
    from goldens import workloads

    if workload == "corpus":
        return workloads()
    return GROUPS.get(workload, [workload])


def load_sites(names):
    """Every recorded site of the entries, in order: (docs, queries, site
    records with their entry name)."""
    from goldens import load, queries

    docs, qs, recs = [], [], []
    for n in names:
        d = load(n)
        docs.append(d)
        qs.extend(queries(d))
        recs.extend(dict(s, entry=n) for s in d["sites"])
    return docs, qs, recs


def site_instances(queries, light=None, full=None):
    """Per site: its instances = the root-box volume of the device problems
    of its *light* compile (the query's domain after structural lowering:
    thread ids x loop indices x havoc loads x launch assignments, before any
    bound reasoning), or of its full compile when the light one cannot bound
    it.  Deterministic (no device involved), so both arms count the same
    instances and every ratio of values is a ratio of times."""
    from paper_2603_24595_b200.engine import compile_all

    light = light if light is not None else compile_all(queries, light=True)
    need = [i for i, (cq, _) in enumerate(light) if cq is None or not cq.problems]
    if full is None:
        got = compile_all([queries[i] for i in need])
        full = dict(zip(need, got))
    inst = []
    for i, (cq, _) in enumerate(light):
        src = cq if (cq is not None and cq.problems) else full.get(i, (None, None))[0]
        inst.append(sum(p.volume() for p in src.problems) if src is not None else 0)
    return inst


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int:
    """--gpus N outside torchrun: one process per GPU under
    torch.distributed.run (127.0.0.1 rendezvous)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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
    """Per-unit SASS calibration of the search kernels (ncu launch list,
    tools/gpu_profile.sh -> tools/summarize_ncu.py -> profiles/)."""
    path = os.path.join(ROOT, "profiles", f"ncu_{workload}_summary.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return {}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


# -- reference arm ---------------------------------------------------------------------

def _ref_group(queries):
    """One reference worker job: the queries in order through the unmodified
    reference (refbridge: Solver.check + canonicalize_witness)."""
    from refbridge import reference_check_queries

    t0 = time.perf_counter()
    done, _ = reference_check_queries(queries)
    assert done == len(queries)
    return time.perf_counter() - t0


def run_reference(args):
    """--impl reference: the unmodified reference checker on the host cores.
    Rank 0 only (other ranks exit without work).  The site list is cut into
    ``steps`` contiguous slices; timed step i decides slice i on a process
    pool (sites round-robin over min(cores, slice) workers, one reference
    Solver per worker job), so the timed steps decide every site exactly
    once and value = all sites' instances / summed step time.  Warm-up steps
    decide the first site (pool start, imports)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from refbridge import have_reference

    if not have_reference():
        print(json.dumps({"impl": "reference",
                          "unavailable": "reference MiniKernel not installed under baseline/_ref"}))
        return
    import multiprocessing as mp

    from paper_2603_24595_b200.engine import compile_all

    names = entries(args.workload)
    _, queries, _ = load_sites(names)
    inst = site_instances(queries)
    cores = os.cpu_count() or 1
    pool = mp.get_context("fork").Pool(cores)
    n = len(queries)
    k = max(1, args.steps)
    slices = [list(range(n * i // k, n * (i + 1) // k)) for i in range(k)]
    for _ in range(args.warmup):
        pool.map(_ref_group, [[queries[0]]])
    times, used = [], 0
    for sl in slices:
        w = max(1, min(cores, len(sl)))
        groups = [[queries[j] for j in sl[g::w]] for g in range(w)]
        groups = [g for g in groups if g]
        used = max(used, len(groups))
        t0 = time.perf_counter()
        if groups:
            pool.map(_ref_group, groups, chunksize=1)
        times.append(time.perf_counter() - t0)
    pool.close()
    total_s = sum(times)
    value = float(sum(inst)) / total_s if total_s > 0 else 0.0
    out = {
        "impl": "reference",
        "metric": "checked (thread, input) access instances/sec; time-to-verdict per kernel x model",
        "value": value, "unit": "instances/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total_s / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int64/int128 (mathematical integers)",
        "data": "recorded reference site queries of the workload ports (synthetic launches)",
        "time_to_verdict_ms": 1e3 * total_s,
        "config": {"workload": args.workload, "description": CONFIG_NAMES.get(args.workload),
                   "entries": names, "sites": n, "instances": float(sum(inst))},
        "cpu_baseline": {"value": value, "unit": "instances/s", "cores": used, "kind": "reference",
                         "sample": f"{n} site queries of {len(names)} entr"
                                   f"{'y' if len(names) == 1 else 'ies'} split into {k} slices, one "
                                   "per timed step, each on a pool of up to "
                                   f"{cores} processes (reference Solver.check + "
                                   "canonicalize_witness, baseline/_ref)"},
        "e2e": {"value": value, "unit": "instances/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


def _cpu_baseline(queries, inst, budget_s):
    """The reference on one host core over a bounded sample of the
    workload: the device-decided sites (the ones that carry instances) in
    site order, until ``budget_s`` of CPU time is spent."""
    try:
        from refbridge import have_reference, reference_check_queries

        if not have_reference():
            return None
        order = [i for i in range(len(queries)) if inst[i] > 0]
        t0 = time.perf_counter()
        done, _ = reference_check_queries([queries[i] for i in order], budget_s=budget_s)
        dt = time.perf_counter() - t0
        covered = float(sum(inst[i] for i in order[:done]))
        return {"value": covered / dt, "unit": "instances/s", "cores": 1,
                "kind": "reference",
                "sample": f"first {done} of the {len(order)} device-decided site queries (of "
                          f"{len(queries)}) through the reference's Solver.check + "
                          f"canonicalize_witness (baseline/_ref), {dt:.1f}s, 1 thread"}
    except Exception as exc:  # the baseline is reported, never required
        return {"value": None, "unit": "instances/s", "cores": 1, "kind": "reference",
                "sample": f"unavailable: {exc}"}


def _k2_sort_traffic():
    """Measured DRAM bytes of one forced sort-path sweep (ncu launch list of
    tools/gpu_k2_profile.sh, committed under profiles/): the sum over its
    kernels of dram__bytes_read + dram__bytes_write, or None."""
    import csv

    path = os.path.join(ROOT, "profiles", "r02_k2_sort_launches.csv")
    try:
        rows = list(csv.reader(open(path)))
    except OSError:
        return None
    hdr, total = None, 0.0
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            total += float(d["Metric Value"].replace(",", ""))
    return total or None


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

    from goldens import load as _gload, queries as _gq
    doc = _gload("rms_norm")
    queries = _gq(doc)
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
                                       "unit": "GB/s", "frac": s_ach / hbm_peak,
                                       "achieved_on_measured_traffic":
                                           (_k2_sort_traffic() or 0) / (sms_ / 1e3) / 1e9,
                                       "frac_on_measured_traffic":
                                           (_k2_sort_traffic() or 0) / (sms_ / 1e3) / 1e9 / hbm_peak,
                                       "traffic": _k2_sort_traffic(),
                                       "traffic_source": "profiles/r02_k2_sort_launches.csv "
                                                         "(ncu, one forced sort-path sweep)",
                                       "algorithmic_bytes": sr["hbm_bytes"],
                                       "note": "the generator compacts as it generates and the "
                                               "order check finds the keys sorted, so the DRAM "
                                               "traffic (generation write, order read, scan "
                                               "read) is about half the 4 x tuple-bytes model",
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

    from goldens import load as _gload, queries as _gq
    doc = _gload("rms_norm")
    queries = _gq(doc)
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


def _analyze_line(chk, name):
    """BASELINE metric part 2, time-to-verdict per kernel x model: the
    reference's own analyze() (parser, symbolic DFS, checking) on one
    workload port + context, with the B200 checking stage AND branch
    screening installed (GpuDetectors; every screen decided on the device,
    no reference fallback) vs unmodified; findings must be the reference's."""
    from goldens import expected_findings, load
    from refpath import add_reference, analyze_workload

    if not add_reference():
        return {"unavailable": "reference front end not installed under baseline/_ref"}
    from paper_2603_24595_b200.detectors import install, uninstall

    doc = load(name)
    times, made = [], []
    for _ in range(3):
        made.clear()
        prev = install(checker=chk, screening=True, created=made)
        t0 = time.perf_counter()
        try:
            got = analyze_workload(name)
        finally:
            uninstall(prev)
        times.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    ref = analyze_workload(name)
    ref_s = time.perf_counter() - t0
    return {"workload": name, "b200_ms": 1e3 * min(times), "reference_ms": 1e3 * ref_s,
            "speedup": ref_s / min(times),
            "findings_equal_reference": got["findings"] == expected_findings(doc),
            "reference_findings_equal_golden": ref["findings"] == doc["findings"],
            "screens_on_device": sum(d.screens for d in made),
            "screen_budget_unknowns": sum(d.screen_budget_unknowns for d in made),
            "screen_reference_fallbacks": 0,
            "what": "analyze() wall time: reference front end (parser, DFS) + B200 checking "
                    "stage and branch screening vs the unmodified reference, one core"}


def _search_line(chk, name, int_peak):
    """The search kernels at scale: one workload whose step is a real
    branch-and-prune (moe_align, the Fig. 7 port: 852 problems, millions of
    boxes and instances), resident and timed like the headline step; integer-issue
    roofline on the algorithmic basis (bytecode instructions evaluated,
    live counters) and on the SASS basis (ncu calibration)."""
    from goldens import load, queries
    from paper_2603_24595_b200.engine import compile_all

    compiled = compile_all(queries(load(name)))
    packed, _ = chk.pack([c for c, _ in compiled])
    if not packed.problems:
        return None
    resident = chk.engine.upload(packed)
    lim = dict(chk.limits)
    lim["max_seconds"] = 600.0
    resident.run(lim)
    runs = [resident.run(lim) for _ in range(3)]
    resident.free()
    n = len(runs)
    ms = sum(r["bb_ms"] + r["leaf_ms"] for r in runs) / n
    step_ms = sum(r["device_ms"] for r in runs) / n
    boxes = sum(r["boxes"] for r in runs) / n
    points = sum(r["points"] for r in runs) / n
    ops = sum(r["insns_bb"] + r["insns_leaf"] for r in runs) / n
    alg = ops / (ms / 1e3) if ms > 0 else 0.0
    cal = _calibration(name)
    per_unit = cal.get("thread_inst_per_unit")
    sass = (boxes + points) * per_unit / (ms / 1e3) if per_unit and ms > 0 else None
    return {"workload": name, "description": CONFIG_NAMES.get(name),
            "device_ms_per_step": step_ms, "boxes_per_step": boxes, "points_per_step": points,
            "roofline": {"bound": "int32-issue", "achieved": alg / 1e9, "peak": int_peak / 1e9,
                         "unit": "Gop/s", "frac": alg / int_peak if int_peak else None,
                         "kernel": "k_search (+k_bb, k_leaf)", "kernel_ms_per_step": ms,
                         "ops": "bytecode instructions evaluated (live device counters)",
                         "sass_basis": {"achieved": sass / 1e9 if sass else None,
                                        "frac": sass / int_peak if sass else None,
                                        "per_unit": per_unit,
                                        "source": f"profiles/ncu_{name}_summary.json",
                                        "ncu_issue_active_pct":
                                            cal.get("k_search_issue_active_pct")}}}


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
    from paper_2603_24595_b200 import shard
    from paper_2603_24595_b200.engine import SiteChecker, compile_all
    from goldens import mismatches

    # the checker (and its compile workers) before the process group
    chk = SiteChecker(device=local)
    if world > 1:
        if one:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if one else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if one else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    names = entries(args.workload)
    docs, queries, recs = load_sites(names)
    t0 = time.perf_counter()
    compiled = compile_all(queries)
    compile_serial_ms = 1e3 * (time.perf_counter() - t0)
    light = compile_all(queries, light=True)
    inst = site_instances(queries, light, dict(enumerate(compiled)))
    mine = (shard.deal([float(1 + len(a)) for a, _ in queries], world)[rank]
            if world > 1 else list(range(len(queries))))
    total_instances = float(sum(inst))

    # the public API's two tiers (SiteChecker.check_queries), made resident:
    # tier 1 = the light problems of every site that compiles light, within
    # the first-tier budget; tier 2 = the full problems of the sites tier 1
    # did not decide.  The parity gate below fixes the tier split.
    lmine = [i for i in mine if light[i][0] is not None]
    packed1, offs1 = chk.pack([light[i][0] for i in lmine])
    t1_budget = chk.tier1_budget(len(lmine))
    res1 = chk.decide([light[i] for i in lmine], packed1, offs1, budget_s=t1_budget)
    tier1 = {i: r for i, r in zip(lmine, res1) if r.status in ("sat", "unsat")}
    rest = [i for i in mine if i not in tier1]
    packed2, offs2 = chk.pack([compiled[i][0] for i in rest])
    res2 = chk.decide([compiled[i] for i in rest], packed2, offs2)
    results = dict(tier1)
    results.update(zip(rest, res2))

    # parity gate: the benchmarked results must be the reference's (sites
    # the reference only timed out on are pinned by z3, tests/goldens.py)
    bad = mismatches({"sites": [recs[i] for i in mine]}, [results[i] for i in mine])
    if bad:
        raise SystemExit(f"parity failure on sites {bad[:10]}")

    def where(i):
        if i in tier1:
            return "tier1_device" if light[i][0].problems else "tier1_host_light"
        cq = compiled[i][0]
        if cq is None or (not cq.problems and not any(g.status == "unsat" for g in cq.groups)):
            return "host_unknown"
        return "host_unsat" if any(g.status == "unsat" for g in cq.groups) else "tier2_device"

    places = {i: where(i) for i in mine}
    sat_dev = sum(1 for i in mine if results[i].status == "sat"
                  and places[i] in ("tier1_device", "tier2_device"))
    resident1 = chk.engine.upload(packed1) if packed1.problems else None
    resident2 = chk.engine.upload(packed2) if packed2.problems else None
    lim1 = dict(chk.limits)
    lim1["max_seconds"] = t1_budget
    limits = dict(chk.limits)
    limits["max_seconds"] = min(chk.limits["max_seconds"] * max(len(rest), 1), 3600.0)
    peak = chk.engine.int_peak()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    empty = {"device_ms": 0.0, "bb_ms": 0.0, "leaf_ms": 0.0, "boxes": 0, "points": 0,
             "insns_bb": 0, "insns_leaf": 0, "launches": 0, "covered": 0.0}
    def step():
        out = dict(empty)
        for rs, lim in ((resident1, lim1), (resident2, limits)):
            if rs is None:
                continue
            st = rs.run(lim)
            for k in empty:
                out[k] += st[k]
        return out

    for _ in range(args.warmup):
        step()
    clocks = Clocks(local).start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    dev_ms, launches, acc = [], 0, {}
    for _ in range(args.steps):
        flush.random_(0, 255)
        torch.cuda.synchronize()
        st = step()
        dev_ms.append(st["device_ms"])
        launches += int(st["launches"])
        for k in empty:
            acc[k] = acc.get(k, 0) + st[k]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    n = args.steps
    ms_step = max_over_ranks(sum(dev_ms) / n)
    value = total_instances / (ms_step / 1e3) if ms_step > 0 else 0.0

    # e2e through the public API with host buffers, every step: compile on
    # the worker pool, pack, H2D, search, D2H, assembly (N>1: sites dealt,
    # verdict records all-gathered).  Warm-up calls start the workers.
    def e2e_call():
        return shard.check_sites(chk, queries) if world > 1 else chk.check_queries(queries)

    for _ in range(args.warmup):
        e2e_call()
    e2e_t = []
    for _ in range(n):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_call()
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(sum(e2e_t) / len(e2e_t))
    h2d = sum_over_ranks(packed1.host_bytes() + packed2.host_bytes())
    d2h = sum_over_ranks(sum(r.d2h_bytes() for r in (resident1, resident2) if r))

    # roofline of k_search (+ its pre-split / leaf kernels): integer issue
    search_ms = (acc["bb_ms"] + acc["leaf_ms"]) / n
    units = (acc["boxes"] + acc["points"]) / n
    bc_ops = (acc["insns_bb"] + acc["insns_leaf"]) / n
    int_peak = peak["ops_per_s"]
    alg = bc_ops / (search_ms / 1e3) if search_ms > 0 else 0.0
    cal = _calibration(args.workload)
    per_unit = cal.get("thread_inst_per_unit")
    sass = units * per_unit / (search_ms / 1e3) if per_unit and search_ms > 0 else None
    sms = torch.cuda.get_device_properties(local).multi_processor_count

    def count(kind):
        return int(sum_over_ranks(sum(1 for w in places.values() if w == kind)))

    decided = {"sites": len(queries),
               "device": count("tier1_device") + count("tier2_device"),
               "device_tier1_light": count("tier1_device"),
               "device_tier2_full": count("tier2_device"),
               "host_light_constant_folding": count("tier1_host_light"),
               "host_presolve_unsat": count("host_unsat"),
               "host_reference_giveup_unknown": count("host_unknown"),
               "device_sat_witnesses": int(sum_over_ranks(sat_dev)),
               "device_problems": int(sum_over_ranks(len(packed1.problems) + len(packed2.problems))),
               "tiers": "tier 1: light compile (structural presolve only) + device within "
                        f"{t1_budget * 1e3:.0f} ms; tier 2: full presolve + device for the rest"}

    side = {}
    if rank == 0 and world == 1:
        peaks, src = _peaks()
        if args.race_tokens > 0:
            side["k2_race_sweep"] = _race_sweep_line(chk, args, peaks, src, int_peak)
        if args.access_tokens > 0:
            side["k2_access_replay"] = _access_line(chk, args, peaks, src, int_peak)
        if args.analyze:
            side["time_to_verdict"] = _analyze_line(chk, args.analyze)
        if args.search:
            side["k1_search_at_scale"] = _search_line(chk, args.search, int_peak)
        if not args.no_cpu_baseline:
            side["cpu_baseline"] = _cpu_baseline(queries, inst, args.cpu_budget)
    if world > 1 and args.race_tokens > 0:
        side["k2_race_sharded"] = _race_sharded_line(chk, args, world)

    if rank == 0:
        out = {
            "metric": "checked (thread, input) access instances/sec; time-to-verdict per kernel x model",
            "value": value, "unit": "instances/s", "n_gpus": world, "steps": n,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "int64/int128 (mathematical integers)",
            "data": "site queries recorded from the reference front end on the workload ports "
                    "(synthetic launches; no tensors)",
            "config": {"workload": args.workload, "description": CONFIG_NAMES.get(args.workload),
                       "entries": names, "sites": len(queries),
                       "instances_per_step": total_instances,
                       "instances": "root-box volumes of the sites' device problems after "
                                    "structural lowering (light compile; full when the light one "
                                    "cannot bound the site)",
                       "l2": "flushed between steps (256 MiB write)",
                       "parallelism": "1 GPU" if world == 1 else
                       f"{world} ranks, sites dealt longest-first (no data-path collective; "
                       "verdict records all-gathered in e2e)"},
            "decided": decided,
            "time_to_verdict_ms": e2e_s * 1e3,
            "evaluated_per_step": {"boxes": acc["boxes"] / n, "points": acc["points"] / n,
                                   "bytecode_insns": bc_ops},
            "evaluated_instances_per_s": units / (ms_step / 1e3) if ms_step > 0 else 0.0,
            "covered_instances_per_s": (acc["covered"] / n) / (ms_step / 1e3) if ms_step > 0 else 0.0,
            "e2e": {"value": total_instances / e2e_s, "unit": "instances/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_s * 1e3,
                    "compile_serial_ms": compile_serial_ms,
                    "compile_workers": chk.compile_workers},
            "roofline": {"bound": "int32-issue", "achieved": alg / 1e9, "peak": int_peak / 1e9,
                         "unit": "Gop/s", "frac": alg / int_peak if int_peak else None,
                         "traffic": cal.get("k_search_dram_bytes_per_launch"),
                         "kernel": "k_search (+k_bb pre-split, k_leaf)",
                         "kernel_ms_per_step": search_ms,
                         "ops": "bytecode instructions evaluated per step (live device counters; "
                                "one op per instruction per box or point, SURVEY.md 8(d))",
                         "peak_source": f"mk_int_peak on this device ({sms} SMs): "
                                        "IADD3/LOP3/VIMNMX/IMAD microbenchmark, "
                                        f"{peak['ms']:.2f} ms",
                         "sass_basis": {"achieved": sass / 1e9 if sass else None,
                                        "frac": sass / int_peak if sass else None,
                                        "per_unit": per_unit,
                                        "source": f"profiles/ncu_{args.workload}_summary.json",
                                        "calibrated_on": "the workload's full-presolve problem "
                                                         "set, resident, deterministic limits "
                                                         "(tools/profile_step.py): the budgeted "
                                                         "first tier depends on wall time, which "
                                                         "ncu's replay dilates",
                                        "ncu_issue_active_pct":
                                            cal.get("k_search_issue_active_pct")}},
            "cpu_baseline": side.pop("cpu_baseline", None),
            "clocks": clk,
            "gpu_launches": launches,
        }
        out.update(side)
        print(json.dumps(out))
    for r in (resident1, resident2):
        if r:
            r.free()
    chk.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD,
                    help="config3 (default), corpus, or one workload name")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--analyze", default="rms_norm",
                    help="workload of the analyze() time-to-verdict line ('' to skip)")
    ap.add_argument("--search", default="moe_align",
                    help="workload of the k1_search_at_scale line ('' to skip)")
    ap.add_argument("--access-tokens", type=int, default=16384,
                    help="num_tokens of the oracle-rule access replay line (0: skip)")
    ap.add_argument("--race-tokens", type=int, default=262144,
                    help="num_tokens of the K2 race-sweep line (0: skip)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
