"""Multi-rank checking on CPU: world_size-2 gloo process groups drive the
corpus deal and the slab split through the test-only host emulation of the
engine (tests/emu/libmk_emu.so); results must equal the single-rank ones and
the reference goldens."""
import os
import socket
import sys

import pytest

from goldens import load, mismatches, queries

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EMU = os.path.join(ROOT, "tests", "emu", "libmk_emu.so")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, names, out_dir):
    import json

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from goldens import load as gload, queries as gqueries
    from paper_2603_24595_b200 import shard
    from paper_2603_24595_b200.engine import SiteChecker

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    chk = SiteChecker(lib_path=EMU, compile_workers=0)
    try:
        if mode == "slab":
            res = [shard.check_slabbed(chk, gqueries(gload(n))) for n in names]
        elif mode == "sites":
            res = [shard.check_sites(chk, gqueries(gload(n))) for n in names]
        else:
            res = shard.check_corpus(chk, [gqueries(gload(n)) for n in names])
        with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fh:
            json.dump([[(r.status, r.witness) for r in rs] for rs in res], fh)
    finally:
        chk.close()
        dist.destroy_process_group()


def _run(mode, names, tmp_path, world=2):
    import json

    import torch.multiprocessing as mp

    port = _free_port()
    mp.spawn(_worker, args=(world, port, mode, names, str(tmp_path)), nprocs=world, join=True)
    outs = [json.load(open(os.path.join(tmp_path, f"rank{r}.json"))) for r in range(world)]
    return outs


class _R:
    def __init__(self, status, witness):
        self.status, self.witness = status, witness


@pytest.mark.parametrize("mode", ["slab", "corpus", "sites"])
def test_two_rank_gloo_matches_goldens(mode, tmp_path):
    names = ["racy", "rms_norm", "moe_align_mixtral"]
    outs = _run(mode, names, tmp_path)
    assert outs[0] == outs[1]                      # every rank holds the full answer
    for name, rs in zip(names, outs[0]):
        assert mismatches(load(name), [_R(s, w) for s, w in rs]) == []


def test_slabs_partition_the_root_box():
    from paper_2603_24595_b200.compiler import Problem
    from paper_2603_24595_b200.shard import slab

    p = Problem(var_names=["a", "b"], lo=[3, 0], hi=[9, 5], maximize=[True, False])
    for world in (1, 2, 3, 4, 7, 8, 16):
        pieces = [slab(p, r, world) for r in range(world)]
        got = sorted(v for q in pieces if q is not None for v in range(q.lo[0], q.hi[0] + 1))
        assert got == list(range(3, 10))
        # rank order is preference order: a is maximised, rank 0 holds the top
        firsts = [q.hi[0] for q in pieces if q is not None]
        assert firsts == sorted(firsts, reverse=True)
        assert all(q.lo[1] == 0 and q.hi[1] == 5 for q in pieces if q is not None)


def test_combine_is_lexicographic_and_conservative():
    from paper_2603_24595_b200.compiler import Problem
    from paper_2603_24595_b200.shard import combine_slabs

    p = Problem(var_names=["a", "b"], lo=[0, 0], hi=[9, 9], maximize=[True, False])
    sat_lo = [("sat", [4, 1])]
    sat_hi = [("sat", [7, 5])]
    unsat = [("unsat", None)]
    unknown = [("unknown", None)]
    assert combine_slabs([p], [sat_lo, sat_hi]) == [("sat", [7, 5])]
    assert combine_slabs([p], [unsat, sat_lo]) == [("sat", [4, 1])]
    assert combine_slabs([p], [unsat, unsat]) == [("unsat", None)]
    assert combine_slabs([p], [unknown, sat_hi]) == [("unknown", None)]


def test_slab_rounds_and_domination():
    from paper_2603_24595_b200.compiler import Problem
    from paper_2603_24595_b200.shard import dominated, slab_rounds

    r = slab_rounds(30.0, 0.25)
    assert abs(sum(r) - 30.0) < 1e-9 and r[:3] == [0.25, 0.5, 1.0]
    assert slab_rounds(0.1, 0.25) == [0.1]
    p = Problem(var_names=["a"], lo=[0], hi=[9], maximize=[False])
    # a model in a better-ordered slab closes the later ones, not the earlier
    assert dominated(p, 1, ["sat", "unknown", "unknown"])
    assert dominated(p, 2, ["unsat", "sat", "unknown"])
    assert not dominated(p, 0, ["unknown", "sat", "unknown"])
    q = Problem(var_names=["a"], lo=[0], hi=[9], maximize=[False], any_model=True)
    assert dominated(q, 0, ["unknown", "sat"])      # feasibility: any model decides


class _StubEngine:
    """Rank 0's slab has a model at once; rank 1's slab never finishes in
    budget (every round ends on the clock)."""

    def __init__(self, rank):
        self.rank, self.calls, self.last_stats = rank, 0, {}

    def solve(self, problems, lim):
        self.calls += 1
        self.last_stats = {"seconds": lim["max_seconds"]}
        if self.rank == 0:
            return [("sat", [p.lo[0]]) for p in problems]
        return [("unknown", None) for _ in problems]


class _StubChecker:
    def __init__(self, rank):
        from paper_2603_24595_b200.compiler import CompiledQuery, Group, Problem

        self.limits = {"max_seconds": 30.0}
        self.engine = _StubEngine(rank)
        p = Problem(var_names=["a"], lo=[0], hi=[99], maximize=[False])
        self.cq = CompiledQuery(witness_names=["a"], order=[("a", "min")],
                                groups=[Group("pending", None, False, problems=[0])],
                                problems=[p], defs={}, free_default={})

    def compile(self, queries):
        return [(self.cq, None) for _ in queries]


def _incumbent_worker(rank, world, port, out_dir):
    import json

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2603_24595_b200 import shard

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        chk = _StubChecker(rank)
        res = shard.check_slabbed(chk, [None])
        with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fh:
            json.dump({"calls": chk.engine.calls, "rounds": chk.last_slab_rounds,
                       "res": [(r.status, r.witness) for r in res]}, fh)
    finally:
        dist.destroy_process_group()


def test_slab_incumbent_exchange_stops_dominated_slab(tmp_path):
    """Rank 1's undecided slab stops after the first exchange: rank 0's
    model precedes every point of it, so the answer is rank 0's model."""
    import json

    import torch.multiprocessing as mp

    mp.spawn(_incumbent_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    outs = [json.load(open(os.path.join(tmp_path, f"rank{r}.json"))) for r in range(2)]
    assert outs[0]["res"] == outs[1]["res"] == [["sat", {"a": 0}]]
    assert outs[1]["calls"] == 1 and outs[0]["rounds"] == outs[1]["rounds"] == 1


def test_deal_balances_and_covers():
    from paper_2603_24595_b200.shard import deal

    costs = [9, 1, 1, 1, 5, 5, 2, 8]
    for world in (1, 2, 3, 8):
        parts = deal(costs, world)
        assert sorted(i for part in parts for i in part) == list(range(len(costs)))
        loads = [sum(costs[i] for i in part) for part in parts]
        assert max(loads) - min(loads) <= max(costs)


def test_record_round_trip_128_bit():
    from paper_2603_24595_b200.compiler import Problem
    from paper_2603_24595_b200.shard import _decode, _encode

    p = Problem(var_names=["x", "y", "z"], lo=[0] * 3, hi=[1] * 3, maximize=[False] * 3)
    vals = [-(1 << 100) - 3, (1 << 64) + 5, -1]
    rec = _encode([p, p], [("sat", vals), ("unknown", None)])
    assert _decode([p, p], rec) == [("sat", vals), ("unknown", None)]


def _race_worker(rank, world, port, out_dir):
    import json

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from paper_2603_24595_b200 import shard
    from paper_2603_24595_b200.native import Engine
    from test_race_sweep import _cases

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    eng = Engine(0, EMU)
    try:
        rows = []
        for name, i, launch, expect, prog in _cases():
            if prog.instances > 400_000:
                continue
            got = shard.race_sweep_sharded(eng, prog)
            rows.append([name, i] + [int(got[k]) for k in
                                      ("tuples", "conflicts", "has_race", "idx_a", "idx_b", "offset")])
        with open(os.path.join(out_dir, f"race{rank}.json"), "w") as fh:
            json.dump(rows, fh)
    finally:
        eng.close()
        dist.destroy_process_group()


def test_race_sweep_sharded_equals_single(tmp_path):
    """K2 across ranks (gloo, world 3, host emulation): every store site's
    sharded sweep equals the single-rank sweep (tuples, conflicts, verdict,
    first pair, offset) on every rank, whether the shards combine in the
    fused form or fall back to the whole-launch sweep."""
    import json

    import torch.multiprocessing as mp

    from paper_2603_24595_b200.native import Engine
    from test_race_sweep import _cases

    world = 3
    port = _free_port()
    mp.spawn(_race_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    outs = [json.load(open(os.path.join(tmp_path, f"race{r}.json"))) for r in range(world)]
    assert outs[0] == outs[1] == outs[2] and outs[0]
    eng = Engine(0, EMU)
    try:
        want = {}
        for name, i, launch, expect, prog in _cases():
            if prog.instances > 400_000:
                continue
            got = eng.race_sweep(prog)
            want[(name, i)] = [int(got[k]) for k in
                               ("tuples", "conflicts", "has_race", "idx_a", "idx_b", "offset")]
    finally:
        eng.close()
    for row in outs[0]:
        assert row[2:] == want[(row[0], row[1])], row
    assert any(row[4] for row in outs[0])      # racy sites among them


def test_combine_detects_boundary_conflict():
    from paper_2603_24595_b200 import shard

    base = {"sorted": 1, "instances": 4, "tuples": 4, "conflicts": 0, "has_race": 0,
            "idx_a": 0, "idx_b": 0, "offset": 0, "off_lo": 0, "nblocks": 1, "have": 1}
    a = dict(base, first_key=1, first_id=0, first_idx=0, last_key=5, last_id=3, last_idx=3)
    b = dict(base, first_key=5, first_id=4, first_idx=4, last_key=9, last_id=7, last_idx=7)
    got = shard.combine_race_shards([a, b])
    assert got["conflicts"] == 1 and got["has_race"] and (got["idx_a"], got["idx_b"]) == (3, 4)
    c = dict(b, first_key=4)
    assert shard.combine_race_shards([a, c]) is None       # out of order across the boundary
    d = dict(b, first_id=3)
    assert shard.combine_race_shards([a, d])["conflicts"] == 0   # same thread
