"""K2 race sweep (include/mk_b200.h mk_race_sweep): concrete replay of every
store site of the reference goldens at a concrete launch.

* sat race sites are replayed at the launch of the reference's canonical
  witness: the sweep must find a race there, and its reported pair must be a
  race by the reference's definition (engine/detectors.py:204-273);
* unsat race sites are replayed at the least launch of the store's path (the
  canonical model of the single-thread path, decided by the engine): no race;
* every sweep equals the pure-Python restatement (race.brute_force) in
  tuples, adjacent conflicts and verdict.

The CPU tests drive the test-only host emulation; the GPU tests the sm_100a
kernels (radix sort + conflict scan in HBM)."""
import os

import pytest

from goldens import load, queries, workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EMU = os.path.join(ROOT, "tests", "emu", "libmk_emu.so")
SKIP = {"moe_align"}   # 121 unsat store sites of one instruction: only its sat site here
_CACHE = {}


def _cases():
    """(workload, site index, launch, expected has_race) for every sweepable
    store site; launches for unsat sites come from the emulated engine."""
    if "cases" in _CACHE:
        return _CACHE["cases"]
    from paper_2603_24595_b200 import race
    from paper_2603_24595_b200.engine import SiteChecker

    chk = SiteChecker(lib_path=EMU, compile_workers=0)
    out = []
    seen = set()
    for name in workloads():
        if name.startswith("rotary_") and name != "rotary_embedding":
            continue
        doc = load(name)
        for i, (s, (a, o)) in enumerate(zip(doc["sites"], queries(doc))):
            if s["site"] != "store_site" or s["verdict"] == "unknown":
                continue
            if name in SKIP and s["verdict"] != "sat":
                continue
            key = (name, s["line"], s["col"], len(a))
            if key in seen:
                continue
            seen.add(key)
            if s["verdict"] == "sat":
                launch = s["witness"]
            else:
                path, _, _ = race.split_race_query(a)
                r = chk.check(path, o)
                if r.status != "sat":
                    continue
                launch = r.witness
            try:
                prog = race.race_program(a, o, launch)
            except race.NotSweepable:
                continue
            out.append((name, i, launch, s["verdict"] == "sat", prog))
    chk.close()
    _CACHE["cases"] = out
    return out


def _check(sweep, name, i, expect, prog):
    from paper_2603_24595_b200 import ir, race

    got = sweep(prog)
    if prog.instances <= 200_000:
        tuples, conflicts, has = race.brute_force(prog)
        assert (got["tuples"], got["conflicts"], bool(got["has_race"])) == \
            (tuples, conflicts, has), (name, i)
    assert bool(got["has_race"]) == expect, (name, i)
    if got["has_race"]:
        a, b = got["pair"]
        for x in (a, b):
            assert all(race._truthy(at, x) for at in prog.path) or prog.n_exist
        assert ir.evaluate(prog.offset, a) == ir.evaluate(prog.offset, b) == got["offset"]
        ids = race.ID_NAMES[3:] if prog.shared else race.ID_NAMES
        assert any(a.get(n, 0) != b.get(n, 0) for n in ids)
        if prog.shared:
            assert all(a.get(n, 0) == b.get(n, 0) for n in race.ID_NAMES[:3])


def test_cases_cover_sat_and_unsat_sites():
    cases = _cases()
    assert any(c[4].n_exist for c in cases)            # existential symbols exercised
    assert sum(1 for c in cases if c[3]) >= 3          # racy x2, moe_align
    assert sum(1 for c in cases if not c[3]) >= 10


def test_emulated_sweep_matches_reference_definition():
    from paper_2603_24595_b200.native import Engine

    eng = Engine(0, EMU)
    for name, i, launch, expect, prog in _cases():
        _check(eng.race_sweep, name, i, expect, prog)


def test_existential_vars_and_exit_pinning():
    """rms_norm's output store: the first loop's exit symbol is pinned to its
    concrete value and its index, which touches neither the offset nor an
    identity, only appears in atoms that hold on the whole box (exact linear
    cancellation after its lattice substitution), so it drops out; the
    instance box is then finite: blocks x threads x iterations."""
    from paper_2603_24595_b200 import race

    doc = load("rms_norm")
    launch = {"BS": 1, "SL": 8, "TC": 8, "blockDim.x": 1024, "blockDim.y": 1, "blockDim.z": 1,
              "gridDim.x": 8, "gridDim.y": 1, "gridDim.z": 1}
    progs = []
    for s, (a, o) in zip(doc["sites"], queries(doc)):
        if s["site"] == "store_site" and s["line"] == 20:
            progs.append(race.race_program(a, o, launch))
    big = max(progs, key=lambda p: p.instances)
    assert big.n_exist == 0 and big.inner == 1
    assert big.instances == 8 * 1024 * 4
    assert not any(n.startswith("idx$0") for n in big.problem.var_names)
    assert "threadIdx.x" in big.problem.var_names and "blockIdx.x" in big.problem.var_names


@pytest.mark.gpu
def test_device_sweep_matches_reference_definition():
    from paper_2603_24595_b200.native import Engine

    eng = Engine(0)
    for name, i, launch, expect, prog in _cases():
        _check(eng.race_sweep, name, i, expect, prog)
    eng.close()


@pytest.mark.gpu
def test_device_sweep_full_launch_rms_norm():
    """Config 1 (rms_norm, Llama-2-7B hidden 4096) output store replayed at
    num_tokens = 4096: 16.8 M accesses sorted in HBM, no race."""
    from paper_2603_24595_b200 import race
    from paper_2603_24595_b200.native import Engine

    doc = load("rms_norm")
    T = 4096
    launch = {"BS": 1, "SL": T, "TC": T, "blockDim.x": 1024, "blockDim.y": 1, "blockDim.z": 1,
              "gridDim.x": T, "gridDim.y": 1, "gridDim.z": 1}
    eng = Engine(0)
    for s, (a, o) in zip(doc["sites"], queries(doc)):
        if s["site"] == "store_site" and s["line"] == 20:
            prog = race.race_program(a, o, launch)
            got = eng.race_sweep(prog)
            assert not got["has_race"] and got["conflicts"] == 0
            assert got["tuples"] in (T * 4, T * 1023 * 4)
    eng.close()


@pytest.mark.gpu
def test_device_sweep_paths_agree():
    """The fused ordered pass (NVRTC-specialised, no tuples in HBM), the
    specialised sort path and the interpreted sort path give the same tuples,
    conflicts and first pair; the fused pass decides the in-order cases and
    hands the out-of-order ones to the radix sort."""
    from paper_2603_24595_b200.native import Engine

    eng = Engine(0)
    keys = ("tuples", "conflicts", "has_race", "idx_a", "idx_b", "offset", "sorted")
    seen_sorted, seen_fused_race = set(), False
    for name, i, launch, expect, prog in _cases():
        runs = []
        for env in ({}, {"MK_RACE_NO_FAST": "1"}, {"MK_NO_JIT": "1"}):
            for k in ("MK_NO_JIT", "MK_RACE_NO_FAST"):
                os.environ.pop(k, None)
            os.environ.update(env)
            try:
                runs.append(eng.race_sweep(prog))
            finally:
                for k in env:
                    os.environ.pop(k, None)
        fast, slow, interp = runs
        assert interp["jit"] == 0 and interp["fused"] == 0 and slow["fused"] == 0
        assert [fast[k] for k in keys] == [slow[k] for k in keys] == [interp[k] for k in keys], \
            (name, i, fast, slow)
        assert fast["fused"] == (1 if fast["sorted"] else 0)
        if fast["tuples"] > 1:
            seen_sorted.add(bool(fast["sorted"]))
        seen_fused_race |= bool(fast["fused"] and fast["has_race"])
    assert seen_sorted == {True, False}
    assert seen_fused_race
    eng.close()


@pytest.mark.gpu
def test_device_shards_combine_to_the_whole_sweep():
    """K2 across GPUs, one device: the launch cut into 2, 3 and 8 contiguous
    instance ranges (what race_sweep_sharded gives each rank), each decided by
    the fused pass, combined exactly (shard.combine_race_shards) equals the
    whole-launch sweep; out-of-order shards report unsorted."""
    from paper_2603_24595_b200 import shard
    from paper_2603_24595_b200.native import Engine

    eng = Engine(0)
    keys = ("tuples", "conflicts", "has_race", "idx_a", "idx_b", "offset")
    combined = 0
    try:
        for name, i, launch, expect, prog in _cases():
            whole = eng.race_sweep(prog)
            for world in (2, 3, 8):
                parts = [eng.race_sweep(prog, *shard.shard_range(prog.instances, r, world))
                         if shard.shard_range(prog.instances, r, world)[1] >
                         shard.shard_range(prog.instances, r, world)[0] else
                         {"sorted": 1, "have": 0, "instances": 0, "tuples": 0, "conflicts": 0,
                          "has_race": 0}
                         for r in range(world)]
                got = shard.combine_race_shards(parts)
                if got is None:
                    assert not whole["sorted"], (name, i, world)
                    continue
                combined += 1
                assert [got[k] for k in keys] == [whole[k] for k in keys], (name, i, world)
    finally:
        eng.close()
    assert combined > 0
