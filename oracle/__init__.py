"""CPU oracle of Powersort (arXiv 2605.27147) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2605_27147_b200``) never imports it and shares no code
with it; ``vmps_oracle.c`` is a plain single-threaded C implementation of the
paper's Alg. 1 with three merge variants (copy-merge, Fig. 1;
Virtual-Memory pages, Sec. 4; Pingpong, Sec. 3).  See ``vmps_oracle.c`` for the passage each
function follows and DESIGN.md for the readings of the paper it takes.

Parity pins: tests/test_oracle.py (brute-force power definition, Python's
stable ``sorted``, golden fixtures, paper bounds).  The VM variant's memory
constants are pinned only in magnitude against Fig. 4:
the paper prints pre-allocated worst-case reserves, the oracle allocates on
demand.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "vmps_oracle.c")
_HDR = os.path.join(_HERE, "vmps_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

U32, U64, F32 = 0, 1, 2
VARIANT_A, VARIANT_B, VARIANT_C, VARIANT_C0 = 0, 1, 2, 3  # copy-merge, virtual-memory, pingpong (+ without last-pop)
KIND_ASC, KIND_DESC, KIND_EXT = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle with gcc -O2 (the paper's flag)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-Wall", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Merge(ctypes.Structure):
    _fields_ = [("i", ctypes.c_uint64), ("j", ctypes.c_uint64), ("k", ctypes.c_uint64),
                ("power", ctypes.c_uint32), ("pad", ctypes.c_uint32)]


MERGE_DTYPE = np.dtype([("i", "<u8"), ("j", "<u8"), ("k", "<u8"), ("power", "<u4"),
                        ("pad", "<u4")])


class _Stats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint64) for f in (
        "n", "runs", "merges", "merge_cost_M", "minrun", "comp_runs", "comp_merge",
        "moves_runs", "moves_merge_out", "moves_staging", "moves_copy", "max_stack",
        "reversed_elems", "extended_runs", "page_elems", "peak_extra_pages",
        "peak_extra_elems", "peak_meta_words", "evictions")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.orc_minrun.restype = ctypes.c_uint32
        _lib.orc_minrun.argtypes = [ctypes.c_uint64]
        for f in (_lib.orc_power, _lib.orc_power_brute):
            f.restype = ctypes.c_uint32
            f.argtypes = [ctypes.c_uint64] * 4
        _lib.orc_page_size.restype = ctypes.c_uint64
        _lib.orc_page_size.argtypes = [ctypes.c_uint64, ctypes.c_uint32]
        _lib.orc_less.restype = ctypes.c_int
        _lib.orc_less.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64]
        _lib.orc_sort.restype = ctypes.c_int
        _lib.orc_sort.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                  ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_uint64, ctypes.c_void_p, ctypes.POINTER(_Stats)]
        _lib.orc_plan.restype = ctypes.c_int
        _lib.orc_plan.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                  ctypes.c_void_p, ctypes.POINTER(_Stats)]
        _lib.orc_set_vm_words.restype = None
        _lib.orc_set_vm_words.argtypes = [ctypes.c_uint32]
        _lib.orc_policy.restype = ctypes.c_int
        _lib.orc_policy.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64,
                                    ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]
    return _lib


def policy(n: int, run_start) -> tuple[np.ndarray, int]:
    """Alg. 1's merge plan over given run starts -> (merges, max stack height)."""
    rs = np.ascontiguousarray(run_start, dtype=np.uint64)
    mg = np.zeros(max(len(rs), 1), MERGE_DTYPE)
    ms = ctypes.c_uint64(0)
    rc = lib().orc_policy(n, rs.ctypes.data, len(rs), mg.ctypes.data, ctypes.byref(ms))
    if rc != 0:
        raise RuntimeError(f"orc_policy failed: {rc}")
    return mg[:max(len(rs) - 1, 0)].copy(), int(ms.value)


def set_vm_words(T: int = 0) -> None:
    """Test hook: page-size word count of variant B (0 = the element's own)."""
    lib().orc_set_vm_words(T)


def minrun(n: int) -> int:
    return int(lib().orc_minrun(n))


def power(n: int, i: int, j: int, k: int) -> int:
    return int(lib().orc_power(n, i, j, k))


def power_brute(n: int, i: int, j: int, k: int) -> int:
    return int(lib().orc_power_brute(n, i, j, k))


def page_size(n: int, T: int) -> int:
    return int(lib().orc_page_size(n, T))


def key_type_of(keys: np.ndarray) -> int:
    if keys.dtype == np.uint32:
        return U32
    if keys.dtype == np.uint64:
        return U64
    if keys.dtype == np.float32:
        return F32
    raise TypeError(f"unsupported key dtype {keys.dtype}")


@dataclass
class Plan:
    run_start: np.ndarray  # uint64[runs]
    run_kind: np.ndarray   # uint8[runs]  (bit0 DESC, bit1 EXT)
    merges: np.ndarray     # MERGE_DTYPE[runs-1], Alg. 1 execution order


def _stats_dict(st: _Stats) -> dict:
    return {f: int(getattr(st, f)) for f, _ in _Stats._fields_}


def _cap(n: int, mr: int) -> int:
    m = mr if mr else minrun(max(n, 1))
    return n // max(m, 1) + 2


def sort(keys: np.ndarray, vals: np.ndarray | None = None, variant: int = VARIANT_A,
         minrun_override: int = 0):
    """Stable Powersort of (keys, vals) -> (keys_out, vals_out, Plan, stats)."""
    kt = key_type_of(keys)
    k = np.ascontiguousarray(keys).copy()
    v = None if vals is None else np.ascontiguousarray(vals, dtype=np.uint32).copy()
    n = k.shape[0]
    cap = _cap(n, minrun_override)
    rs = np.zeros(cap, np.uint64)
    rk = np.zeros(cap, np.uint8)
    mg = np.zeros(cap, MERGE_DTYPE)
    st = _Stats()
    kp = k.view(np.uint32 if kt == F32 else k.dtype)
    rc = lib().orc_sort(kt, kp.ctypes.data, None if v is None else v.ctypes.data, n, variant,
                        minrun_override, rs.ctypes.data, rk.ctypes.data, cap, mg.ctypes.data,
                        ctypes.byref(st))
    if rc != 0:
        raise RuntimeError(f"orc_sort failed: {rc}")
    r = st.runs
    plan = Plan(rs[:r].copy(), rk[:r].copy(), mg[:max(r - 1, 0)].copy())
    return k, v, plan, _stats_dict(st)


def plan(keys: np.ndarray, minrun_override: int = 0):
    """Plan only (ExtractRun + Power + Alg. 1 without merging) -> (Plan, stats)."""
    kt = key_type_of(keys)
    k = np.ascontiguousarray(keys)
    n = k.shape[0]
    cap = _cap(n, minrun_override)
    rs = np.zeros(cap, np.uint64)
    rk = np.zeros(cap, np.uint8)
    mg = np.zeros(cap, MERGE_DTYPE)
    st = _Stats()
    kp = k.view(np.uint32 if kt == F32 else k.dtype)
    rc = lib().orc_plan(kt, kp.ctypes.data, n, minrun_override, rs.ctypes.data, rk.ctypes.data,
                        cap, mg.ctypes.data, ctypes.byref(st))
    if rc != 0:
        raise RuntimeError(f"orc_plan failed: {rc}")
    r = st.runs
    return Plan(rs[:r].copy(), rk[:r].copy(), mg[:max(r - 1, 0)].copy()), _stats_dict(st)


def sort_records(records: np.ndarray) -> np.ndarray:
    """Stable lexicographic sort of n records of w unsigned 32-bit words, word 0
    most significant -- the paper's blob data types (arrays of 30
    ints ordered lexicographically; ``ptr`` sorts pointers to such arrays).
    Returns the permutation (int64): the plain definition, Python's stable
    ``sorted`` of the indices by the tuple of words (equal records keep their
    input order).  Pinned in tests/test_oracle.py against the Powersort oracle
    for one-word records and by brute force on tiny inputs."""
    r = np.ascontiguousarray(records, dtype=np.uint32)
    if r.ndim != 2:
        raise ValueError("records must be an (n, words) array")
    rows = [tuple(int(x) for x in row) for row in r]
    return np.array(sorted(range(len(rows)), key=lambda i: rows[i]), dtype=np.int64)
