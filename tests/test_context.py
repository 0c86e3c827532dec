"""Context inference (paper_2603_24595_b200.context)
against the reference's own infer_context (context.py:315-495) on generated
invocation logs: identical canonical context JSON, identical errors."""
import json
import random

import pytest

from refpath import add_reference

HAVE_REF = add_reference()


def _log(seed, kernel="k"):
    rnd = random.Random(seed)
    bss = rnd.sample([1, 2, 3, 4, 5, 8], rnd.randint(2, 3))
    sls = rnd.sample([1, 7, 16, 17, 128, 512], rnd.randint(2, 3))
    hidden = rnd.choice([4096, 7168, 8192])
    off = rnd.choice([0, 1, -1])
    lines = []
    for bs in bss:
        for sl in sls:
            tc = bs * sl
            lines.append(json.dumps({"record": "run", "batch_size": bs, "seq_len": sl}))
            args = [
                {"kind": "tensor", "shape": [tc, hidden], "itemsize": 2, "dtype": "f16"},
                {"kind": "tensor", "shape": [tc + off, hidden], "itemsize": 2, "dtype": "f16"},
                {"kind": "tensor", "shape": [hidden], "itemsize": 2, "dtype": "f16"},
                {"kind": "tensor", "shape": [bs, 64], "itemsize": 4, "dtype": "i32",
                 "int_min": rnd.choice([0, 1]), "int_max": rnd.randint(0, 4 * sl)},
                {"kind": "scalar", "value": rnd.choice([1e-6, 1e-5])},
                {"kind": "scalar", "value": sl * rnd.choice([1, 2])},
                {"kind": "scalar", "value": rnd.randint(0, 50)},
            ]
            lines.append(json.dumps({"record": "call", "kernel": kernel, "args": args}))
            if rnd.random() < 0.3:
                lines.append(json.dumps({"record": "call", "kernel": "other", "args": args[:2]}))
    return "\n".join(lines) + "\n"


def _both(text, kernel):
    from minikernel.context import ContextError, context_to_json, infer_context, parse_log

    from paper_2603_24595_b200.context import infer_context_json

    try:
        want = context_to_json(infer_context(parse_log(text, "log"), kernel))
    except ContextError as exc:
        want = ("error", str(exc))
    try:
        got = infer_context_json(text, kernel, "log")
    except ContextError as exc:
        got = ("error", str(exc))
    return got, want


@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
@pytest.mark.parametrize("seed", range(40))
def test_generated_logs_match_reference(seed):
    got, want = _both(_log(seed), "k")
    assert got == want


@pytest.mark.skipif(not HAVE_REF, reason="reference front end not available")
def test_errors_match_reference():
    text = _log(3)
    for kernel in ("missing", "other"):
        got, want = _both(text, kernel)
        assert got == want and got[0] == "error"
