"""Command line (paper_2603_24595_b200.cli; the reference's specified CLI,
SPEC.md:633-687): exit codes 0 / 1 / 2, the reference's report format from
``analyze``, context inference from an invocation log, the oracle-rule race
replay.  Device commands are GPU tests; argument / file errors and ``infer``
run on the CPU."""
import json
import os
import subprocess
import sys

import pytest

from goldens import expected_findings, load
from refpath import ROOT, add_reference

HAVE_REF = add_reference()
W = os.path.join(ROOT, "workloads")


def _cli(*args):
    env = dict(os.environ)
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    p = subprocess.run([sys.executable, "-m", "paper_2603_24595_b200", *args], cwd=ROOT,
                       capture_output=True, text=True, env=env, timeout=600)
    return p.returncode, p.stdout, p.stderr


def test_missing_kernel_is_operational_error(tmp_path):
    rc, _, err = _cli("analyze", "--kernel", str(tmp_path / "nope.mk"))
    assert rc == 2 and "error" in err


@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
def test_bad_context_path_is_operational_error():
    rc, _, _ = _cli("analyze", "--kernel", os.path.join(W, "racy", "kernel.mk"),
                    "--context", "/nonexistent/ctx.json")
    assert rc == 2


@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
def test_infer_recovers_laws_from_a_nine_run_log(tmp_path):
    """SPEC.md acceptance 5 shape: BS in {1,3,5} x SL in {1,7,17}, input
    [TC, 7168] f16, weight [7168], eps 1e-6 -> Linear(TC), Invariant(7168),
    Invariant(eps)."""
    lines = []
    for bs in (1, 3, 5):
        for sl in (1, 7, 17):
            tc = bs * sl
            lines.append(json.dumps({"record": "run", "batch_size": bs, "seq_len": sl}))
            lines.append(json.dumps({"record": "call", "kernel": "k", "args": [
                {"kind": "tensor", "shape": [tc, 7168], "itemsize": 2, "dtype": "f16"},
                {"kind": "tensor", "shape": [7168], "itemsize": 2, "dtype": "f16"},
                {"kind": "scalar", "value": 1e-6}]}))
    log = tmp_path / "runs.jsonl"
    log.write_text("\n".join(lines) + "\n")
    out = tmp_path / "ctx.json"
    rc, _, err = _cli("infer", "--log", str(log), "--kernel", "k", "--out", str(out))
    assert rc == 0, err
    ctx = json.loads(out.read_text())
    laws = {(a["position"], c["feature"]): c for a in ctx["args"] for c in a["constraints"]}
    assert laws[(0, "dim0")]["law"] == "linear" and laws[(0, "dim0")]["basis"] == "TC"
    assert laws[(0, "dim1")]["law"] == "invariant" and laws[(0, "dim1")]["value"] == 7168
    assert laws[(2, "value")]["law"] == "invariant"


@pytest.mark.gpu
@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
def test_analyze_prints_the_reference_report():
    rc, out, err = _cli("analyze", "--kernel", os.path.join(W, "racy", "kernel.mk"),
                        "--context", os.path.join(W, "racy", "ctx.json"))
    assert rc == 1, err
    assert json.loads(out)["findings"] == expected_findings(load("racy"))


@pytest.mark.gpu
@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
def test_races_finds_the_missing_barrier():
    rc, out, err = _cli("races", "--kernel", os.path.join(W, "racy_rw", "kernel.mk"),
                        "--context", os.path.join(W, "racy_rw", "ctx.json"),
                        "--launch", "BS=2,SL=64")
    assert rc == 1, err
    doc = json.loads(out)
    assert doc["has_race"] and doc["racy_granules"] == 64
    assert (doc["first"]["write"]["kind"], doc["first"]["other"]["kind"]) == ("write", "read")


@pytest.mark.gpu
@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
def test_corpus_one_line_per_entry():
    rc, out, err = _cli("corpus", os.path.join(W, "racy"), os.path.join(W, "rms_norm"))
    assert rc == 1, err
    rows = [json.loads(x) for x in out.splitlines() if x.strip()]
    assert [os.path.basename(r["entry"]) for r in rows] == ["racy", "rms_norm"]
    assert rows[1]["findings"] == expected_findings(load("rms_norm"))


@pytest.mark.gpu
@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
def test_replay_confirms_the_narrowing_and_deref_witnesses():
    for name, kind in (("silu_and_mul", "IntegerOverflow"), ("copy_blocks", "InvalidDeref")):
        rc, out, err = _cli("replay", "--kernel", os.path.join(W, name, "kernel.mk"),
                            "--context", os.path.join(W, name, "ctx.json"))
        assert rc == 0, err
        rows = [json.loads(line) for line in out.splitlines() if line.startswith("{")]
        assert rows and all(r["status"] in ("confirmed", "confirmed-expression") for r in rows)
        assert any(r["kind"] == kind and r["status"] == "confirmed" for r in rows)
