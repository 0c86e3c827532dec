"""ctypes binding of ``libmk_b200.so`` (C ABI in ``include/mk_b200.h``).

The product path loads ONLY the in-tree CUDA library built by
``__graft_entry__.build()``; there is no CPU fallback.  A missing library or
a host without a CUDA device raises :class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libmk_b200.so"
DEFAULT_LIB = os.path.join(HERE, LIB_NAME)

MK_UNSAT, MK_SAT, MK_UNKNOWN = 0, 1, 2
MK_PF_NARROW = 1
MK_PF_ANY = 2
STATUS_NAME = {MK_UNSAT: "unsat", MK_SAT: "sat", MK_UNKNOWN: "unknown"}

EXPORTS = ("mk_abi_version", "mk_device_count", "mk_ctx_create", "mk_ctx_destroy",
           "mk_last_error", "mk_site_eval", "mk_set_upload", "mk_set_eval", "mk_set_free",
           "mk_race_sweep")


class NativeUnavailable(RuntimeError):
    """The CUDA checking engine cannot run here."""


# -- ABI structs (must match include/mk_b200.h) ------------------------------------

I128 = np.dtype([("lo", "<u8"), ("hi", "<i8")])
INSN = np.dtype([("op", "<u2"), ("dst", "<u2"), ("a", "<u2"), ("b", "<u2"),
                 ("c", "<u2"), ("pad", "<u2")])
PROBLEM = np.dtype([("nvars", "<i4"), ("ninsn", "<i4"), ("nregs", "<i4"), ("natoms", "<i4"),
                    ("nconst", "<i4"), ("nrows", "<i4"), ("var_off", "<i4"),
                    ("insn_off", "<i4"), ("const_off", "<i4"), ("atom_off", "<i4"),
                    ("row_off", "<i4"), ("flags", "<i4"), ("maxmask", "<u8")])
ROW = np.dtype([("rel", "<i4"), ("nterms", "<i4"), ("term_off", "<i4"), ("group", "<i4"),
                ("c0", I128)])
ROW_TERM = np.dtype([("var", "<i4"), ("pad0", "<i4"), ("pad1", "<i8"), ("coef", I128)])
assert PROBLEM.itemsize == 56 and INSN.itemsize == 12 and ROW.itemsize == 32
assert ROW_TERM.itemsize == 32 and I128.itemsize == 16


class ProblemSet(ctypes.Structure):
    _fields_ = [("nprob", ctypes.c_int32), ("nvar_total", ctypes.c_int32),
                ("ninsn_total", ctypes.c_int32), ("nconst_total", ctypes.c_int32),
                ("natom_total", ctypes.c_int32), ("nrow_total", ctypes.c_int32),
                ("nterm_total", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("probs", ctypes.c_void_p), ("var_lo", ctypes.c_void_p),
                ("var_hi", ctypes.c_void_p), ("insns", ctypes.c_void_p),
                ("consts", ctypes.c_void_p), ("atom_regs", ctypes.c_void_p),
                ("atom_masks", ctypes.c_void_p), ("rows", ctypes.c_void_p),
                ("row_terms", ctypes.c_void_p)]


class Limits(ctypes.Structure):
    _fields_ = [("max_rounds", ctypes.c_int64), ("max_boxes", ctypes.c_int64),
                ("max_seconds", ctypes.c_double), ("split_k", ctypes.c_int32),
                ("chunk", ctypes.c_int32), ("leaf_volume", ctypes.c_int64),
                ("unit_stack", ctypes.c_int64)]


class Stats(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_int64), ("boxes", ctypes.c_int64),
                ("leaves", ctypes.c_int64), ("points", ctypes.c_int64),
                ("covered", ctypes.c_double), ("seconds", ctypes.c_double),
                ("bb_ms", ctypes.c_double), ("leaf_ms", ctypes.c_double),
                ("insns_bb", ctypes.c_int64), ("insns_leaf", ctypes.c_int64),
                ("device_ms", ctypes.c_double), ("launches", ctypes.c_int64),
                ("steps", ctypes.c_int64), ("strategy", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class RaceProg(ctypes.Structure):
    _fields_ = [("set", ProblemSet), ("off_reg", ctypes.c_int32), ("shared", ctypes.c_int32),
                ("id_var", ctypes.c_int32 * 6), ("n_exist", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("begin", ctypes.c_uint64), ("end", ctypes.c_uint64)]


class RaceResult(ctypes.Structure):
    _fields_ = [("instances", ctypes.c_uint64), ("tuples", ctypes.c_uint64),
                ("conflicts", ctypes.c_uint64), ("has_race", ctypes.c_int32),
                ("sort_bits", ctypes.c_int32), ("idx_a", ctypes.c_uint64),
                ("idx_b", ctypes.c_uint64), ("offset", ctypes.c_int64),
                ("gen_ms", ctypes.c_double), ("sort_ms", ctypes.c_double),
                ("scan_ms", ctypes.c_double), ("hbm_bytes", ctypes.c_uint64),
                ("jit", ctypes.c_int32), ("sorted", ctypes.c_int32),
                ("fused", ctypes.c_int32), ("have", ctypes.c_int32),
                ("first_key", ctypes.c_uint64), ("first_id", ctypes.c_uint64),
                ("first_idx", ctypes.c_uint64), ("last_key", ctypes.c_uint64),
                ("last_id", ctypes.c_uint64), ("last_idx", ctypes.c_uint64),
                ("off_lo", ctypes.c_int64), ("nblocks", ctypes.c_uint64),
                ("sort_passes", ctypes.c_int32), ("pad", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class AccessProg(ctypes.Structure):
    _fields_ = [("off_reg", ctypes.c_int32), ("n_exist", ctypes.c_int32),
                ("id_var", ctypes.c_int32 * 6), ("id_fixed", ctypes.c_int64 * 6),
                ("write", ctypes.c_int32), ("shared", ctypes.c_int32),
                ("granule", ctypes.c_int32), ("tuples", ctypes.c_int32),
                ("kbase", ctypes.c_uint64), ("span", ctypes.c_uint64), ("off_lo", ctypes.c_int64)]


class AccessInput(ctypes.Structure):
    _fields_ = [("set", ProblemSet), ("progs", ctypes.c_void_p),
                ("grid", ctypes.c_int64 * 3), ("block", ctypes.c_int64 * 3),
                ("key_bits", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("nkeys", ctypes.c_uint64)]


class AccessResult(ctypes.Structure):
    _fields_ = [("instances", ctypes.c_uint64), ("tuples", ctypes.c_uint64),
                ("racy", ctypes.c_uint64), ("has_race", ctypes.c_int32),
                ("misaligned", ctypes.c_int32), ("slot_a", ctypes.c_uint64),
                ("slot_b", ctypes.c_uint64), ("gen_ms", ctypes.c_double),
                ("sort_ms", ctypes.c_double), ("scan_ms", ctypes.c_double),
                ("fast", ctypes.c_int32), ("jit", ctypes.c_int32),
                ("sort_passes", ctypes.c_int32), ("pad", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


assert ctypes.sizeof(AccessProg) == 120 and ctypes.sizeof(AccessResult) == 88
assert ctypes.sizeof(RaceProg) == 160 and ctypes.sizeof(RaceResult) == 176


def _bind(lib: ctypes.CDLL) -> ctypes.CDLL:
    lib.mk_abi_version.restype = ctypes.c_int
    lib.mk_device_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
    lib.mk_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    lib.mk_ctx_destroy.argtypes = [ctypes.c_void_p]
    lib.mk_last_error.argtypes = [ctypes.c_void_p]
    lib.mk_last_error.restype = ctypes.c_char_p
    lib.mk_site_eval.argtypes = [ctypes.c_void_p, ctypes.POINTER(ProblemSet),
                                 ctypes.POINTER(Limits), ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.POINTER(Stats)]
    lib.mk_set_upload.argtypes = [ctypes.c_void_p, ctypes.POINTER(ProblemSet),
                                  ctypes.POINTER(ctypes.c_void_p)]
    lib.mk_set_eval.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Limits),
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Stats)]
    lib.mk_set_free.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    lib.mk_race_sweep.argtypes = [ctypes.c_void_p, ctypes.POINTER(RaceProg),
                                  ctypes.POINTER(RaceResult)]
    lib.mk_access_sweep.argtypes = [ctypes.c_void_p, ctypes.POINTER(AccessInput),
                                    ctypes.POINTER(AccessResult)]
    if hasattr(lib, "mk_sort_pairs_u64"):
        lib.mk_sort_pairs_u64.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_int32)]
    if hasattr(lib, "mk_int_peak"):       # device library only (not the test emulator)
        lib.mk_int_peak.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_double)]
    return lib


_LIBS = {}


def load_library(path: Optional[str] = None) -> ctypes.CDLL:
    path = os.path.abspath(path or DEFAULT_LIB)
    lib = _LIBS.get(path)
    if lib is not None:
        return lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = _bind(ctypes.CDLL(path))
    if lib.mk_abi_version() != 1:
        raise NativeUnavailable(f"{path}: ABI version mismatch")
    _LIBS[path] = lib
    return lib


# -- packing ---------------------------------------------------------------------------

def _i128_array(values: Sequence[int]) -> np.ndarray:
    a = np.zeros(len(values), dtype=I128)
    if len(values):
        try:
            # the common case: every value fits int64 (two's complement lo
            # word, sign-extended hi word)
            v64 = np.asarray(values, dtype=np.int64)
        except OverflowError:
            a["lo"] = [v & 0xFFFFFFFFFFFFFFFF for v in values]
            a["hi"] = [v >> 64 for v in values]
        else:
            a["lo"] = v64.view(np.uint64)
            a["hi"] = v64 >> 63
    return a


def _i128_value(lo: int, hi: int) -> int:
    return (int(hi) << 64) | int(lo)


class PackedSet:
    """Host-side arrays of one ``mk_problem_set`` (kept alive while in use)."""

    def __init__(self, problems) -> None:
        self.problems = list(problems)
        P = len(self.problems)
        # per-problem header columns first, then the flat arrays: one numpy
        # assignment per column (per-element structured-array writes made
        # packing a third of the caller's time in a streamed batch)
        cols = {k: [] for k in ("nvars", "ninsn", "nregs", "natoms", "nconst", "nrows", "var_off",
                                "insn_off", "const_off", "atom_off", "row_off", "flags", "maxmask")}
        lo, hi, consts, atom_regs, atom_masks = [], [], [], [], []
        insns = []
        rows, terms = [], []
        for p in self.problems:
            cols["nvars"].append(p.nvars)
            cols["ninsn"].append(len(p.insns))
            cols["nregs"].append(max(p.nregs, 1))
            cols["natoms"].append(len(p.atom_regs))
            cols["nconst"].append(len(p.consts))
            cols["nrows"].append(len(p.rows))
            cols["var_off"].append(len(lo))
            cols["insn_off"].append(len(insns))
            cols["const_off"].append(len(consts))
            cols["atom_off"].append(len(atom_regs))
            cols["row_off"].append(len(rows))
            m = 0
            for k, mx in enumerate(p.maximize):
                if mx:
                    m |= 1 << k
            cols["maxmask"].append(m)
            cols["flags"].append((MK_PF_NARROW if getattr(p, "narrow", False) else 0) |
                                 (MK_PF_ANY if getattr(p, "any_model", False) else 0))
            lo.extend(p.lo)
            hi.extend(p.hi)
            insns.extend(p.insns)
            consts.extend(p.consts)
            atom_regs.extend(p.atom_regs)
            atom_masks.extend(p.atom_masks)
            for row in p.rows:
                rel, c0, tl = row[:3]
                rows.append((rel, len(tl), len(terms), row[3] if len(row) > 3 else 0, c0))
                terms.extend(tl)
        self.probs = np.zeros(P, dtype=PROBLEM)
        if P:
            for k, v in cols.items():
                self.probs[k] = np.asarray(v, dtype=PROBLEM[k])
        self.var_lo = _i128_array(lo)
        self.var_hi = _i128_array(hi)
        self.insns = np.zeros(len(insns), dtype=INSN)
        if insns:
            arr = np.asarray(insns, dtype=np.int64)
            self.insns["op"] = arr[:, 0]
            self.insns["dst"] = arr[:, 1]
            self.insns["a"] = arr[:, 2]
            self.insns["b"] = arr[:, 3]
            self.insns["c"] = arr[:, 4]
        self.consts = _i128_array(consts)
        self.atom_regs = np.asarray(atom_regs, dtype=np.int32)
        self.atom_masks = np.asarray(atom_masks, dtype=np.uint64)
        self.rows = np.zeros(len(rows), dtype=ROW)
        if rows:
            arr = np.asarray([r[:4] for r in rows], dtype=np.int64)
            self.rows["rel"] = arr[:, 0]
            self.rows["nterms"] = arr[:, 1]
            self.rows["term_off"] = arr[:, 2]
            self.rows["group"] = arr[:, 3]
            self.rows["c0"] = _i128_array([r[4] for r in rows])
        self.terms = np.zeros(len(terms), dtype=ROW_TERM)
        if terms:
            self.terms["var"] = np.asarray([t[0] for t in terms], dtype=np.int32)
            self.terms["coef"] = _i128_array([t[1] for t in terms])
        self.nvar_total = len(lo)
        self.struct = ProblemSet(
            P, len(lo), len(insns), len(consts), len(atom_regs), len(rows), len(terms), 0,
            self.probs.ctypes.data, self.var_lo.ctypes.data, self.var_hi.ctypes.data,
            self.insns.ctypes.data, self.consts.ctypes.data, self.atom_regs.ctypes.data,
            self.atom_masks.ctypes.data, self.rows.ctypes.data, self.terms.ctypes.data)

    def host_bytes(self) -> int:
        return sum(a.nbytes for a in (self.probs, self.var_lo, self.var_hi, self.insns,
                                      self.consts, self.atom_regs, self.atom_masks,
                                      self.rows, self.terms))


class Engine:
    """One device context of the checking engine."""

    def __init__(self, device: int = 0, lib_path: Optional[str] = None) -> None:
        self.lib = load_library(lib_path)
        n = ctypes.c_int(0)
        self.lib.mk_device_count(ctypes.byref(n))
        if n.value <= device:
            raise NativeUnavailable(f"no CUDA device {device} (found {n.value})")
        ctx = ctypes.c_void_p()
        rc = self.lib.mk_ctx_create(device, ctypes.byref(ctx))
        if rc != 0:
            raise NativeUnavailable(f"mk_ctx_create({device}) failed: {rc}")
        self.ctx = ctx
        self.device = device
        self.last_stats: Optional[dict] = None

    def close(self) -> None:
        if getattr(self, "ctx", None):
            self.lib.mk_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve_packed(self, packed: PackedSet, limits: Optional[dict] = None
                     ) -> List[Tuple[str, Optional[List[int]]]]:
        lim = Limits(0, 0, 0.0, 0, 0, 0, 0)
        for k, v in (limits or {}).items():
            setattr(lim, k, v)
        P = len(packed.problems)
        status = np.zeros(max(P, 1), dtype=np.int32)
        point = np.zeros(max(packed.nvar_total, 1), dtype=I128)
        st = Stats()
        rc = self.lib.mk_site_eval(self.ctx, ctypes.byref(packed.struct), ctypes.byref(lim),
                                   status.ctypes.data, point.ctypes.data, ctypes.byref(st))
        if rc != 0:
            msg = self.lib.mk_last_error(self.ctx)
            raise RuntimeError(f"mk_site_eval failed ({rc}): {msg.decode() if msg else ''}")
        self.last_stats = st.as_dict()
        out: List[Tuple[str, Optional[List[int]]]] = []
        for i, p in enumerate(packed.problems):
            s = STATUS_NAME[int(status[i])]
            if s == "sat":
                off = int(packed.probs[i]["var_off"])
                vals = [_i128_value(point[off + k]["lo"], point[off + k]["hi"])
                        for k in range(p.nvars)]
                out.append((s, vals))
            else:
                out.append((s, None))
        return out

    def solve(self, problems, limits: Optional[dict] = None):
        return self.solve_packed(PackedSet(problems), limits)

    # -- race sweep (K2) -----------------------------------------------------------

    def race_sweep(self, prog, begin: int = 0, end: int = 0) -> dict:
        """Concrete race replay of one store at one launch
        (paper_2603_24595_b200.race.RaceProgram -> mk_race_sweep); with
        ``end`` > 0 only instances [begin, end) (a shard of the launch)."""
        packed = PackedSet([prog.problem])
        rp = RaceProg()
        rp.begin = int(begin)
        rp.end = int(end)
        rp.set = packed.struct
        rp.off_reg = prog.off_reg
        rp.shared = 1 if prog.shared else 0
        for i, v in enumerate(prog.id_var):
            rp.id_var[i] = v
        rp.n_exist = prog.n_exist
        out = RaceResult()
        rc = self.lib.mk_race_sweep(self.ctx, ctypes.byref(rp), ctypes.byref(out))
        if rc != 0:
            msg = self.lib.mk_last_error(self.ctx)
            raise RuntimeError(f"mk_race_sweep failed ({rc}): {msg.decode() if msg else ''}")
        res = out.as_dict()
        if res["has_race"]:
            res["pair"] = (prog.decode(res["idx_a"]), prog.decode(res["idx_b"]))
        return res

    def access_sweep(self, problems, progs, grid, block, key_bits, nkeys=0) -> dict:
        """Oracle-semantics race sweep of several accesses at one launch
        (paper_2603_24595_b200.replay -> mk_access_sweep).  ``progs`` is a
        list of dicts with the mk_access_prog fields."""
        packed = PackedSet(problems)
        arr = (AccessProg * len(progs))()
        for a, d in zip(arr, progs):
            for k, v in d.items():
                if k in ("id_var", "id_fixed"):
                    for i, x in enumerate(v):
                        getattr(a, k)[i] = x
                else:
                    setattr(a, k, v)
        inp = AccessInput()
        inp.set = packed.struct
        inp.progs = ctypes.cast(arr, ctypes.c_void_p)
        for i in range(3):
            inp.grid[i] = int(grid[i])
            inp.block[i] = int(block[i])
        inp.key_bits = int(key_bits)
        inp.nkeys = int(nkeys)
        out = AccessResult()
        rc = self.lib.mk_access_sweep(self.ctx, ctypes.byref(inp), ctypes.byref(out))
        if rc != 0:
            msg = self.lib.mk_last_error(self.ctx)
            raise RuntimeError(f"mk_access_sweep failed ({rc}): {msg.decode() if msg else ''}")
        return out.as_dict()

    def sort_pairs(self, keys: np.ndarray, vals: np.ndarray, bits: int = 64,
                   force: bool = False) -> dict:
        """The K2 HBM sort on host arrays (uint64, sorted in place):
        mk_sort_pairs_u64; returns the device time and digit passes."""
        assert keys.dtype == np.uint64 and vals.dtype == np.uint64 and keys.shape == vals.shape
        keys = np.ascontiguousarray(keys)
        vals = np.ascontiguousarray(vals)
        ms, passes = ctypes.c_double(), ctypes.c_int32()
        rc = self.lib.mk_sort_pairs_u64(self.ctx, keys.ctypes.data, vals.ctypes.data, keys.size,
                                        bits, int(force), ctypes.byref(ms), ctypes.byref(passes))
        if rc != 0:
            msg = self.lib.mk_last_error(self.ctx)
            raise RuntimeError(f"mk_sort_pairs_u64 failed ({rc}): {msg.decode() if msg else ''}")
        return {"keys": keys, "vals": vals, "ms": ms.value, "passes": passes.value}

    def int_peak(self) -> dict:
        """Measured INT32 issue rate of this device (mk_int_peak): integer
        thread-instructions per second of the IADD3/LOP3/VIMNMX/IMAD
        microbenchmark, the denominator of the evaluator's roofline."""
        ops, ms = ctypes.c_double(), ctypes.c_double()
        rc = self.lib.mk_int_peak(self.ctx, ctypes.byref(ops), ctypes.byref(ms))
        if rc != 0:
            msg = self.lib.mk_last_error(self.ctx)
            raise RuntimeError(f"mk_int_peak failed ({rc}): {msg.decode() if msg else ''}")
        return {"ops_per_s": ops.value, "ms": ms.value}

    # -- device-resident sets ------------------------------------------------------

    def upload(self, packed: PackedSet) -> "ResidentSet":
        h = ctypes.c_void_p()
        rc = self.lib.mk_set_upload(self.ctx, ctypes.byref(packed.struct), ctypes.byref(h))
        if rc != 0:
            msg = self.lib.mk_last_error(self.ctx)
            raise RuntimeError(f"mk_set_upload failed ({rc}): {msg.decode() if msg else ''}")
        return ResidentSet(self, packed, h)


class ResidentSet:
    """A problem set kept in HBM; ``run`` decides it again without any
    host-to-device copy (only verdicts and points come back)."""

    def __init__(self, engine: Engine, packed: PackedSet, handle) -> None:
        self.engine = engine
        self.packed = packed
        self.handle = handle
        P = len(packed.problems)
        self.status = np.zeros(max(P, 1), dtype=np.int32)
        self.point = np.zeros(max(packed.nvar_total, 1), dtype=I128)

    def run(self, limits: Optional[dict] = None) -> dict:
        lim = Limits(0, 0, 0.0, 0, 0, 0, 0)
        for k, v in (limits or {}).items():
            setattr(lim, k, v)
        st = Stats()
        e = self.engine
        rc = e.lib.mk_set_eval(e.ctx, self.handle, ctypes.byref(lim), self.status.ctypes.data,
                               self.point.ctypes.data, ctypes.byref(st))
        if rc != 0:
            msg = e.lib.mk_last_error(e.ctx)
            raise RuntimeError(f"mk_set_eval failed ({rc}): {msg.decode() if msg else ''}")
        return st.as_dict()

    def d2h_bytes(self) -> int:
        return self.status.nbytes + self.point.nbytes

    def free(self) -> None:
        if self.handle:
            self.engine.lib.mk_set_free(self.engine.ctx, self.handle)
            self.handle = None
