"""The C-ABI library loads without a GPU and exports every entry point that
include/mk_b200.h declares (no compute calls here)."""
import os
import re
import subprocess

from refpath import ROOT

HEADER = os.path.join(ROOT, "include", "mk_b200.h")
LIB = os.path.join(ROOT, "paper_2603_24595_b200", "libmk_b200.so")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(mk_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = _declared()
    for fn in ("mk_abi_version", "mk_device_count", "mk_ctx_create", "mk_ctx_destroy",
               "mk_last_error", "mk_site_eval"):
        assert fn in names


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (mk_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert missing == []


def test_library_loads_and_reports_abi_without_gpu():
    from paper_2603_24595_b200 import native

    lib = native.load_library(LIB)
    assert lib.mk_abi_version() == 1
    import ctypes
    n = ctypes.c_int(-1)
    lib.mk_device_count(ctypes.byref(n))
    assert n.value >= 0


def test_product_has_no_cpu_engine():
    """The package never loads the test-only emulator."""
    from paper_2603_24595_b200 import native

    assert native.DEFAULT_LIB.endswith("libmk_b200.so")
    src = open(os.path.join(ROOT, "paper_2603_24595_b200", "native.py")).read()
    assert "mk_emu" not in src
