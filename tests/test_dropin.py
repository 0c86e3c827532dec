"""End-to-end drop-in parity: the reference's own analyze() with its checking
stage swapped for GpuDetectors must produce the reference's findings array
bit for bit (engine/report.py:41-51, :109-140)."""
import os

import pytest

from goldens import expected_findings, load, workloads
from refpath import ROOT, add_reference, analyze_workload

HAVE_REF = add_reference()
EMU = os.path.join(ROOT, "tests", "emu", "libmk_emu.so")


def _run(name, checker, screening=False, created=None):
    from paper_2603_24595_b200.detectors import install, uninstall

    prev = install(checker=checker, screening=screening, created=created)
    try:
        return analyze_workload(name)
    finally:
        uninstall(prev)


@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
@pytest.mark.parametrize("screening", [False, True])
@pytest.mark.parametrize("name", ["racy", "rms_norm", "fused_add_rms_norm", "copy_blocks", "silu_and_mul",
                                  "float_branch", "rms_norm_unknown_path", "copy_blocks_unknown_path"])
def test_dropin_emulated(name, screening):
    from paper_2603_24595_b200.engine import SiteChecker

    chk = SiteChecker(lib_path=EMU)
    try:
        doc = _run(name, chk, screening)
    finally:
        chk.close()
    assert doc["findings"] == expected_findings(load(name))
    assert doc["coverage"] == "complete"


@pytest.mark.gpu
@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
@pytest.mark.parametrize("screening", [False, True])
@pytest.mark.parametrize("name", workloads())
def test_dropin_gpu(name, screening):
    """Findings with the checking stage on the B200, and with the executor's
    branch screening (engine/executor.py:489-492) on it as well."""
    from paper_2603_24595_b200.engine import SiteChecker

    chk = SiteChecker(device=0)
    made = []
    try:
        doc = _run(name, chk, screening, made)
    finally:
        chk.close()
    assert doc["findings"] == expected_findings(load(name))
    assert doc["coverage"] == "complete"
    if screening:
        # every branch screen decided on the device: no budget cut-offs (and
        # there is no reference fallback to hide one)
        assert made and sum(d.screens for d in made) > 0
        assert sum(d.screen_budget_unknowns for d in made) == 0
