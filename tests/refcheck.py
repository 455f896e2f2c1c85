"""Test-side references that are independent of both oracle/ and the CUDA path.

- stable_sorted: Python's built-in stable ``sorted`` with an explicit order key.
- f32 order key: written with ``math`` predicates (reading R5).
- cartesian_postorder: the merge plan derived from the Cartesian tree of the
  boundary powers, computed by recursive minimum splitting --
  a different derivation from Alg. 1's stack simulation.
- natural-run checks, entropy.
"""
from __future__ import annotations

import math
import struct

import numpy as np


def f32_order_key(bits: int):
    x = struct.unpack("<f", struct.pack("<I", int(bits)))[0]
    if math.isnan(x):
        return (1, 0.0, 0)
    return (0, x, 0 if math.copysign(1.0, x) < 0 else 1)


def order_key_fn(dtype):
    if dtype == np.float32:
        return f32_order_key
    return int


def stable_sorted(keys: np.ndarray, vals: np.ndarray | None = None):
    """(keys, vals) stably sorted by the key order (vals default: original index)."""
    n = len(keys)
    kb = keys.view(np.uint32) if keys.dtype == np.float32 else keys
    kf = order_key_fn(keys.dtype)
    idx = sorted(range(n), key=lambda t: kf(kb[t]))
    idx = np.array(idx, dtype=np.int64)
    v = np.arange(n, dtype=np.uint32) if vals is None else vals
    return keys[idx], v[idx]


def less(dtype, a, b) -> bool:
    kf = order_key_fn(dtype)
    return kf(a) < kf(b)


def check_runs(keys: np.ndarray, run_start, run_kind, minrun: int):
    """Check run starts/kinds against the ExtractRun definition (R3)."""
    n = len(keys)
    kb = keys.view(np.uint32) if keys.dtype == np.float32 else keys
    lt = lambda x, y: less(keys.dtype, kb[x], kb[y])
    rs = [int(x) for x in run_start] + [n]
    assert rs[0] == 0 or n == 0
    for t in range(len(rs) - 1):
        s, e = rs[t], rs[t + 1]
        assert s < e
        desc = s + 1 < n and lt(s + 1, s)
        nat = s + 1
        if desc:
            nat = s + 2
            while nat < n and lt(nat, nat - 1):
                nat += 1
        else:
            while nat < n and not lt(nat, nat - 1):
                nat += 1
        if nat - s < minrun:
            assert e == min(n, s + minrun), (t, s, e, nat)
            kind = (1 if desc else 0) | 2
        else:
            assert e == nat, (t, s, e, nat)
            kind = 1 if desc else 0
        assert int(run_kind[t]) == kind, (t, int(run_kind[t]), kind)


def cartesian_postorder(n: int, run_start, power_fn):
    """Merge records (i, j, k, p) as the post-order of the Cartesian tree (min at root)."""
    rs = [int(x) for x in run_start] + [n]
    r = len(rs) - 1
    if r <= 1:
        return []
    pw = [None] + [power_fn(n, rs[t - 1], rs[t], rs[t + 1]) for t in range(1, r)]
    out = []
    stack = [(1, r - 1, False)]  # iterative post-order over boundary index ranges
    while stack:
        lo, hi, done = stack.pop()
        if lo > hi:
            continue
        t = min(range(lo, hi + 1), key=lambda u: pw[u])
        if done:
            out.append((rs[lo - 1], rs[t], rs[hi + 1], pw[t]))
            continue
        stack.append((lo, hi, True))
        stack.append((t + 1, hi, False))
        stack.append((lo, t - 1, False))
    return out


def entropy(lengths) -> float:
    n = float(sum(lengths))
    return sum((l / n) * math.log2(n / l) for l in lengths)


def read_golden(path):
    d = {"merge": []}
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        k, *v = line.split()
        if k == "merge":
            d["merge"].append(tuple(int(x) for x in v))
        elif k.startswith("keys_"):
            d["keys"] = np.array([int(x) for x in v], dtype={"u32": np.uint32, "u64": np.uint64}[k[5:]])
        else:
            d[k] = [int(x) for x in v]
    return d


def read_table(path, sep=None):
    rows = []
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        rows.append([c.split() for c in line.split("|")] if sep else line.split())
    return rows
