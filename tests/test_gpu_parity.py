"""GPU parity: every reference query of every workload, decided by the
sm_100a engine through the C ABI, must give the reference's verdict and
canonical witness bit for bit (engine/detectors.py + engine/report.py)."""
import pytest

from goldens import load, mismatches, queries, workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def checker():
    from paper_2603_24595_b200.engine import SiteChecker

    chk = SiteChecker(device=0)
    yield chk
    chk.close()


@pytest.mark.parametrize("name", workloads())
def test_batch_parity(checker, name):
    doc = load(name)
    results = checker.check_queries(queries(doc))
    assert mismatches(doc, results) == []


@pytest.mark.parametrize("name", ["racy", "rms_norm"])
def test_single_query_parity(checker, name):
    doc = load(name)
    qs = queries(doc)
    results = [checker.check(*q) for q in qs]
    assert mismatches(doc, results) == []


def test_engine_loaded_from_tree():
    from paper_2603_24595_b200 import native

    lib = native.load_library()
    assert native.DEFAULT_LIB in [p for p in native._LIBS]
    assert lib.mk_abi_version() == 1
