"""Oracle-semantics race replay (paper_2603_24595_b200.replay,
include/mk_b200.h mk_access_sweep): read-write and cross-instruction races
with barrier epochs over a concrete launch (SURVEY.md 8(f)
row 2).  Non-parity: the reference ships no such oracle, so the check is the
pure-Python restatement of the specification's rule (oracle/access_oracle.py)
on the same recorded accesses: race verdict, racy granule count and the
first race's pair must be identical.

The accesses come from the reference's own analyze() with GpuDetectors
recording every executed load / store (install(recorders=...)).  CPU tests
drive the test-only host emulation; the GPU tests the sm_100a sweep."""
import os

import pytest

from refpath import ROOT, add_reference, analyze_workload

HAVE_REF = add_reference()
EMU = os.path.join(ROOT, "tests", "emu", "libmk_emu.so")
_REC = {}


def _recorded(name):
    """(access records, origin_of) of one analyze() run of a workload."""
    if name in _REC:
        return _REC[name]
    from paper_2603_24595_b200.detectors import install, uninstall
    from paper_2603_24595_b200.engine import SiteChecker

    chk = SiteChecker(lib_path=EMU, compile_workers=0)
    recs = []
    prev = install(checker=chk, recorders=recs)
    try:
        analyze_workload(name)
    finally:
        uninstall(prev)
        chk.close()
    accesses = [a for d in recs for a in d.accesses]
    _REC[name] = (accesses, recs[0].table.origin_of)
    return _REC[name]


def _launch(accesses, origin_of, pins):
    """A concrete launch (replay.launch_model, decided by the emulated engine)."""
    from paper_2603_24595_b200 import replay
    from paper_2603_24595_b200.engine import SiteChecker

    chk = SiteChecker(lib_path=EMU, compile_workers=0)
    try:
        return replay.launch_model(chk, accesses, origin_of, pins)
    finally:
        chk.close()


CASES = [
    # race probe: shared s[tx % 4] (same-instruction WW, epoch 0) then a
    # barrier and a read of s[0] (epoch 1: no RW race), global t[bx*8+tx]
    # and t[0] from every thread (cross-instruction WW on t[0])
    ("racy", {"BS": 2, "SL": 3}, True),
    # rms_norm (config 1): shared reduction buffer and per-token output
    ("rms_norm", {"BS": 1, "SL": 2}, None),
    ("fused_add_rms_norm", {"BS": 1, "SL": 2}, None),
    # missing barrier: buf[tx] stored, buf[(tx + 1) % 32] read in the same
    # epoch (a read-write race the reference's twin check cannot see)
    ("racy_rw", {"BS": 2, "SL": 40}, True),
    # fused-MoE kernels (Mixtral-8x7B): shared counters across barriers,
    # data-dependent (havoc) indices as existential symbols
    ("moe_align_mixtral", {"BS": 1, "SL": 1}, None),
    ("topk_softmax", {"BS": 1, "SL": 1}, None),
]


def _compare(engine, name, pins, expect):
    from oracle import access_oracle
    from paper_2603_24595_b200 import replay

    accesses, origin_of = _recorded(name)
    launch = _launch(accesses, origin_of, pins)
    got = replay.replay_races(engine, accesses, origin_of, launch)
    accs, progs, key_bits, skipped = replay.build(accesses, origin_of, launch)
    grid = [launch[d] for d in replay.DIMS[:3]]
    block = [launch[d] for d in replay.DIMS[3:]]
    has, racy, first = access_oracle.sweep(accs, grid, block)
    assert got.accesses == len(accs) and got.accesses > 0
    assert (got.has_race, got.racy) == (has, racy), (name, got.has_race, got.racy, has, racy)
    if expect is not None:
        assert got.has_race == expect
    if has:
        _, head, other = first
        w, o = got.first["write"], got.first["other"]
        assert w["kind"] == "write"
        assert (accs[head[1]].record.line, accs[other[1]].record.line) == (w["line"], o["line"])
        assert w["thread"] != o["thread"]
        assert w["region"] == o["region"]
        if accs[head[1]].record.shared:
            assert w["epoch"] == o["epoch"] and w["thread"][:3] == o["thread"][:3]
    return got


@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
def test_recorder_sees_reads_writes_and_epochs():
    accesses, _ = _recorded("racy")
    kinds = {(a.line, a.kind) for a in accesses}
    assert (8, "write") in kinds and (11, "read") in kinds and (13, "write") in kinds
    shared = [a for a in accesses if a.shared]
    assert {a.epoch for a in shared} == {0, 1}


@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
@pytest.mark.parametrize("name,pins,expect", CASES)
def test_emulated_replay_matches_oracle_rule(name, pins, expect):
    from paper_2603_24595_b200.native import Engine

    eng = Engine(0, EMU)
    try:
        got = _compare(eng, name, pins, expect)
    finally:
        eng.close()
    if name == "racy":
        # the first race is the shared store s[tx % 4] (region order puts
        # shared:s before the tensor), not the barrier-separated read
        assert got.first["write"]["region"] == "shared:s"
        assert got.first["other"]["kind"] == "write"


@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
def test_barrier_separates_shared_epochs():
    """Without barrier epochs the reads of s[0] (racy, line 11) would race
    with the stores of line 8; with them the only shared races are the
    stores' own (4 granules per block)."""
    import copy

    from oracle import access_oracle
    from paper_2603_24595_b200 import replay

    accesses, origin_of = _recorded("racy")
    launch = _launch(accesses, origin_of, {"BS": 1, "SL": 1})
    grid = [launch[d] for d in replay.DIMS[:3]]
    block = [launch[d] for d in replay.DIMS[3:]]
    accs, _, _, _ = replay.build(accesses, origin_of, launch)
    _, racy, first = access_oracle.sweep(accs, grid, block)
    flat = copy.deepcopy(accesses)
    for r in flat:
        r.epoch = 0
    accs2, _, _, _ = replay.build(flat, origin_of, launch)
    _, racy_flat, _ = access_oracle.sweep(accs2, grid, block)
    shared = lambda f: f[0][0] == 0  # noqa: E731  (region rank 0 = shared:s)
    assert shared(first) and racy == 4 + 1       # s[0..3] and t[0]
    assert racy_flat == racy                     # s[0] already racy by the stores


@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
def test_missing_barrier_read_write_race_beyond_reference():
    """racy_rw: the reference reports nothing (its DataRace query pairs a
    store only with its own twin, engine/detectors.py:204-232); the oracle
    replay finds the read of a neighbour's slot racing with its store."""
    from paper_2603_24595_b200 import replay
    from paper_2603_24595_b200.native import Engine

    assert analyze_workload("racy_rw")["findings"] == []
    accesses, origin_of = _recorded("racy_rw")
    launch = _launch(accesses, origin_of, {"BS": 1, "SL": 32})
    eng = Engine(0, EMU)
    try:
        got = replay.replay_races(eng, accesses, origin_of, launch)
    finally:
        eng.close()
    assert got.has_race and got.racy == 32
    w, o = got.first["write"], got.first["other"]
    assert (w["kind"], o["kind"], w["line"], o["line"]) == ("write", "read", 11, 13)
    assert w["epoch"] == o["epoch"] == 0


@pytest.mark.gpu
@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
@pytest.mark.parametrize("name,pins,expect", CASES)
def test_device_replay_matches_oracle_rule(name, pins, expect):
    from paper_2603_24595_b200.native import Engine

    eng = Engine(0)
    try:
        _compare(eng, name, pins, expect)
    finally:
        eng.close()


@pytest.mark.gpu
@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
def test_device_replay_equals_emulation_at_scale():
    """rms_norm at num_tokens 512 (2 M instances per access): device and
    host emulation agree on every count and on the first race."""
    from paper_2603_24595_b200 import replay
    from paper_2603_24595_b200.native import Engine

    accesses, origin_of = _recorded("rms_norm")
    launch = _launch(accesses, origin_of, {"BS": 1, "SL": 512})
    dev, emu = Engine(0), Engine(0, EMU)
    try:
        a = replay.replay_races(dev, accesses, origin_of, launch)
        b = replay.replay_races(emu, accesses, origin_of, launch)
    finally:
        dev.close()
        emu.close()
    assert (a.has_race, a.racy, a.instances, a.tuples) == (b.has_race, b.racy, b.instances, b.tuples)
    assert a.first == b.first
    assert a.fast and not a.has_race             # race-free: the owner-table pass decides


@pytest.mark.gpu
@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
@pytest.mark.parametrize("name,pins,expect", CASES)
def test_device_fast_and_sort_paths_agree(name, pins, expect):
    """The owner-table pass and the radix-sort path reach the same verdict;
    a racy launch always ends on the sort path (canonical first pair)."""
    from paper_2603_24595_b200 import replay
    from paper_2603_24595_b200.native import Engine

    accesses, origin_of = _recorded(name)
    launch = _launch(accesses, origin_of, pins)
    eng = Engine(0)
    try:
        a = replay.replay_races(eng, accesses, origin_of, launch)
        os.environ["MK_ACCESS_NO_FAST"] = "1"
        try:
            b = replay.replay_races(eng, accesses, origin_of, launch)
        finally:
            os.environ.pop("MK_ACCESS_NO_FAST", None)
        os.environ["MK_NO_JIT"] = "1"       # the interpreted generator, both paths
        try:
            c = replay.replay_races(eng, accesses, origin_of, launch)
        finally:
            os.environ.pop("MK_NO_JIT", None)
    finally:
        eng.close()
    assert (a.has_race, a.instances, a.tuples) == (b.has_race, b.instances, b.tuples) == \
        (c.has_race, c.instances, c.tuples)
    assert a.fast == (not a.has_race) and not b.fast
    if a.has_race:
        assert (a.racy, a.first) == (b.racy, b.first) == (c.racy, c.first)
