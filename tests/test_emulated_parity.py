"""CPU parity of the compiler + search logic: the test-only host emulation of
the engine (same evaluation core, serial driver) must reproduce every
reference verdict and canonical witness."""
import os

import pytest

from goldens import load, mismatches, queries, workloads

EMU = os.path.join(os.path.dirname(os.path.abspath(__file__)), "emu", "libmk_emu.so")


@pytest.fixture(scope="module")
def emu_checker():
    from paper_2603_24595_b200.engine import SiteChecker

    chk = SiteChecker(device=0, lib_path=EMU)
    yield chk
    chk.close()


@pytest.mark.parametrize("name", [w for w in workloads() if w != "moe_align" and not w.startswith("paged_attention")])
def test_emulated_parity(emu_checker, name):
    doc = load(name)
    assert mismatches(doc, emu_checker.check_queries(queries(doc))) == []


def test_emulated_parity_moe_align_sample(emu_checker):
    doc = load("moe_align")
    # every sat site plus a stride of the unsat ones keeps the CPU suite short
    keep = [i for i, s in enumerate(doc["sites"]) if s["verdict"] != "unsat" or i % 9 == 0]
    sub = dict(doc, sites=[doc["sites"][i] for i in keep])
    assert mismatches(sub, emu_checker.check_queries(queries(sub))) == []


def test_emulated_parity_paged_attention_sample(emu_checker):
    """paged_attention_v1 needs ~4e8 boxes on the GPU; the host emulation
    checks the sites its serial driver decides within the CPU-suite budget."""
    doc = load("paged_attention_v1")
    keep = [i for i, s in enumerate(doc["sites"]) if s["site"] == "arithmetic_site"]
    sub = dict(doc, sites=[doc["sites"][i] for i in keep])
    assert mismatches(sub, emu_checker.check_queries(queries(sub))) == []
