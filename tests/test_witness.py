"""Witness replay (paper_2603_24595_b200.witness; SPEC.md:573-631
replay_witness): every sat overflow / out-of-bounds / deref witness the
reference produced is confirmed at expression level and over the full
launch it names (every thread swept on the engine), and a launch just below
the canonical witness is not confirmed."""
import os

import pytest

from goldens import load, queries, workloads
from refpath import ROOT

EMU = os.path.join(ROOT, "tests", "emu", "libmk_emu.so")


def _sat_sites(names):
    for name in names:
        doc = load(name)
        for s, (a, o) in zip(doc["sites"], queries(doc)):
            if s["verdict"] == "sat" and s["site"] != "store_site":
                yield name, s, a, o


def _threads(launch):
    n = 1
    for d in ("gridDim.x", "gridDim.y", "gridDim.z", "blockDim.x", "blockDim.y", "blockDim.z"):
        n *= launch.get(d, 1)
    return n


def test_small_launch_witnesses_confirmed_emulated():
    from paper_2603_24595_b200 import witness as W
    from paper_2603_24595_b200.native import Engine

    eng = Engine(0, EMU)
    seen = 0
    for name, s, a, o in _sat_sites(["copy_blocks", "moe_align_mixtral", "moe_align"]):
        if _threads(W.launch_of(s["witness"], o)) > 1 << 16:
            continue
        r = W.replay_witness(eng, a, o, s["witness"])
        assert r.status in ("confirmed", "confirmed-expression"), (name, s["line"], r)
        if r.status == "confirmed":
            assert 1 <= r.violating_threads <= r.candidates
            seen += 1
    assert seen >= 6
    eng.close()


@pytest.mark.gpu
def test_every_sat_witness_confirmed_on_device():
    from paper_2603_24595_b200 import witness as W
    from paper_2603_24595_b200.native import Engine

    eng = Engine(0)
    full = 0
    for name, s, a, o in _sat_sites(workloads()):
        r = W.replay_witness(eng, a, o, s["witness"])
        assert r.status in ("confirmed", "confirmed-expression"), (name, s["line"], r)
        full += r.status == "confirmed"
    assert full >= 20
    eng.close()


@pytest.mark.gpu
def test_one_token_below_the_witness_is_not_confirmed():
    """rms_norm (config 1): the canonical IO witness is num_tokens = 524289
    (blockIdx.x * 4096 passes 2^31 - 1 first there); at 524288 tokens no
    thread of the launch overflows."""
    from paper_2603_24595_b200 import witness as W
    from paper_2603_24595_b200.native import Engine

    eng = Engine(0)
    doc = load("rms_norm")
    for s, (a, o) in zip(doc["sites"], queries(doc)):
        if s["verdict"] != "sat" or s["site"] != "arithmetic_site":
            continue
        w = dict(s["witness"])
        assert W.replay_witness(eng, a, o, w).status == "confirmed"
        t = w["TC"] - 1
        w.update({"SL": t, "TC": t, "gridDim.x": t, "blockIdx.x": t - 1})
        r = W.replay_witness(eng, a, o, w)
        assert r.status == "not-confirmed" and not r.expression, r
    eng.close()
