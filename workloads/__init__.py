"""Seeded synthetic inputs shaped like BASELINE.json's five configs.

Shared by tests, smoke() and bench.py.  This module holds none of the
method's arithmetic (no run detection, powers or merging): it only draws
random numbers and shapes them with library primitives (torch.sort).  The
recipes follow SURVEY 8(d) / readings R12-R14:

  cfg1  n=2^20 u32, uniform random permutation of 0..n-1 (seed 1), no payload
  cfg2  n=2^24 u32 + u32 payload (= index); run lengths uniform [1, 2 sqrt(n)],
        values i.i.d. uniform u32, each run sorted ascending
  cfg3  n=2^26 u64 keys in 0..15 + payload; run lengths uniform [1, 2 sqrt(n)],
        each run sorted, 10% of runs reversed (non-increasing with plateaus)
  cfg4  n=2^28 f32 normal(0,1), 'Timsort-drag' run lengths (reading R13), +0.0
        and -0.0 injected at rate 2^-10 each, each run sorted (value, then -0
        before +0)
  cfg5  n=2^30 per shard u32 + payload (= global index mod 2^32); segments of
        length 1 + Geom0(1/4096); half i.i.d. uniform unsorted, half sorted
        ascending, 5% of those reversed

Every generator takes ``n`` so tests can draw the same shapes at small sizes.
Randomness: a torch.Generator on the target device seeded with ``seed``
(the oracle always sorts a host copy of exactly the tensor the GPU sorts,
so cross-device bit-equality of the generator is not required).
"""
from __future__ import annotations

import math

import torch

CONFIGS = {
    1: dict(n=1 << 20, key="u32", vals=False, desc="n=2^20 u32 random permutation (seed 1)"),
    2: dict(n=1 << 24, key="u32", vals=True, desc="n=2^24 u32+u32 random runs, len U[1,2sqrt n]"),
    3: dict(n=1 << 26, key="u64", vals=True, desc="n=2^26 u64 keys in 0..15 + u32, 10% runs reversed"),
    4: dict(n=1 << 28, key="f32", vals=False, desc="n=2^28 f32 normal, Timsort-drag runs, +-0"),
    5: dict(n=1 << 30, key="u32", vals=True, desc="n=2^30/GPU u32+u32 mixture, geometric runs mean 4096"),
}


def _gen(device, seed: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def _u32_from_i64(x: torch.Tensor) -> torch.Tensor:
    """int64 values in [0, 2^32) -> uint32 tensor (bit-preserving)."""
    return x.to(torch.int32).view(torch.uint32)


def _uniform_u32_i64(n: int, g: torch.Generator, device) -> torch.Tensor:
    return torch.randint(0, 1 << 32, (n,), generator=g, device=device, dtype=torch.int64)


def _segments_uniform(n: int, maxlen: int, g, device) -> torch.Tensor:
    """Run lengths uniform in [1, maxlen], the last one truncated to sum to n."""
    est = max(4, int(2.2 * n / (maxlen + 1)) + 16)
    while True:
        lens = torch.randint(1, maxlen + 1, (est,), generator=g, device=device, dtype=torch.int64)
        cs = torch.cumsum(lens, 0)
        if int(cs[-1]) >= n:
            break
        est *= 2
    k = int(torch.searchsorted(cs, torch.tensor([n], device=device)).item())
    lens = lens[: k + 1].clone()
    lens[k] -= int(cs[k]) - n
    return lens[lens > 0]


def _seg_ids(lens: torch.Tensor) -> torch.Tensor:
    return torch.repeat_interleave(torch.arange(lens.numel(), device=lens.device), lens)


def _sort_within_segments(low: torch.Tensor, seg: torch.Tensor) -> torch.Tensor:
    """Permutation that orders elements by (segment, low) stably (low < 2^32)."""
    comp = (seg << 32) | low
    return torch.sort(comp, stable=True).indices


def drag_lengths(m: int) -> list[int]:
    """Reading R13 of the garbled 'Timsort-drag' rule: R(m) = [m] for m <= 3,
    else with h = floor((m+1)/3): R(h) ++ R(h-1) ++ [m - 2h + 1] (zero-length
    parts dropped).  Iterative to avoid deep recursion."""
    out: list[int] = []
    stack = [("R", m)]
    while stack:
        tag, x = stack.pop()
        if tag == "L" or x <= 3:
            if x > 0:
                out.append(x)
            continue
        h = (x + 1) // 3
        stack.append(("L", x - 2 * h + 1))
        stack.append(("R", h - 1))
        stack.append(("R", h))
    return out


def cfg1(n: int = 1 << 20, seed: int = 1, device="cpu"):
    g = _gen(device, seed)
    keys = torch.randperm(n, generator=g, device=device, dtype=torch.int64)
    return _u32_from_i64(keys), None


def cfg2(n: int = 1 << 24, seed: int = 2, device="cpu"):
    g = _gen(device, seed)
    maxlen = max(1, int(2 * math.isqrt(n)))
    lens = _segments_uniform(n, maxlen, g, device)
    vals = _uniform_u32_i64(n, g, device)
    perm = _sort_within_segments(vals, _seg_ids(lens))
    keys = _u32_from_i64(vals[perm])
    return keys, _u32_from_i64(torch.arange(n, device=device, dtype=torch.int64))


def cfg3(n: int = 1 << 26, seed: int = 3, device="cpu"):
    g = _gen(device, seed)
    maxlen = max(1, int(2 * math.isqrt(n)))
    lens = _segments_uniform(n, maxlen, g, device)
    vals = torch.randint(0, 16, (n,), generator=g, device=device, dtype=torch.int64)
    seg = _seg_ids(lens)
    rev = torch.rand(lens.numel(), generator=g, device=device) < 0.10
    low = torch.where(rev[seg], 15 - vals, vals)
    perm = _sort_within_segments(low, seg)
    keys = vals[perm].to(torch.uint64) if hasattr(torch, "uint64") else vals[perm]
    return keys, _u32_from_i64(torch.arange(n, device=device, dtype=torch.int64))


def cfg4(n: int = 1 << 28, seed: int = 4, device="cpu"):
    g = _gen(device, seed)
    lens = torch.tensor(drag_lengths(n), dtype=torch.int64, device=device)
    x = torch.randn(n, generator=g, device=device, dtype=torch.float64).to(torch.float32)
    u = torch.rand(n, generator=g, device=device)
    x = torch.where(u < 2.0 ** -10, torch.zeros_like(x), x)                    # +0.0
    x = torch.where((u >= 2.0 ** -10) & (u < 2.0 ** -9), torch.full_like(x, -0.0), x)  # -0.0
    seg = _seg_ids(lens)
    # sort each run by (value, -0.0 before +0.0): stable sort by the sign
    # tiebreak, then stable sort by (segment, value)
    neg_first = (~torch.signbit(x)).to(torch.int64)
    p1 = torch.sort(neg_first, stable=True).indices
    x1, seg1 = x[p1], seg[p1]
    p2 = torch.sort(x1.to(torch.float64) + 0.0, stable=True).indices
    x2, seg2 = x1[p2], seg1[p2]
    p3 = torch.sort(seg2, stable=True).indices
    return x2[p3].contiguous(), None


def cfg5(n: int = 1 << 30, seed: int = 5, device="cpu", rank: int = 0):
    g = _gen(device, seed * 1000003 + rank)
    p = 1.0 / 4096
    est = int(n * p * 1.3) + 64
    lens = torch.empty(est, dtype=torch.float64, device=device).geometric_(p, generator=g)
    lens = lens.to(torch.int64)
    cs = torch.cumsum(lens, 0)
    while int(cs[-1]) < n:
        more = torch.empty(est, dtype=torch.float64, device=device).geometric_(p, generator=g).to(torch.int64)
        lens = torch.cat([lens, more])
        cs = torch.cumsum(lens, 0)
    k = int(torch.searchsorted(cs, torch.tensor([n], device=device)).item())
    lens = lens[: k + 1].clone()
    lens[k] -= int(cs[k]) - n
    lens = lens[lens > 0]
    nseg = lens.numel()
    vals = _uniform_u32_i64(n, g, device)
    sorted_seg = torch.rand(nseg, generator=g, device=device) < 0.5
    rev_seg = sorted_seg & (torch.rand(nseg, generator=g, device=device) < 0.05)
    seg = _seg_ids(lens)
    local = torch.arange(n, device=device, dtype=torch.int64)
    low = torch.where(sorted_seg[seg], torch.where(rev_seg[seg], (1 << 32) - 1 - vals, vals), local)
    del local
    perm = _sort_within_segments(low, seg)
    del low, seg
    keys = _u32_from_i64(vals[perm])
    del vals, perm
    base = rank * n
    idx = (torch.arange(n, device=device, dtype=torch.int64) + base) & 0xFFFFFFFF
    return keys, _u32_from_i64(idx)


GENERATORS = {1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4, 5: cfg5}


# ---- the paper's own workload ----
PAPER_N = 10 ** 7
PAPER_S = (2, 10 ** 2, 10 ** 3, 10 ** 4, 10 ** 5, 10 ** 6)


def paper_input(S: int, kind: str = "int", seed: int = 0, N: int = PAPER_N, device="cpu"):
    """One input of the paper's sweep: length n ~ U[9N/10, N]; every integer
    uniform in [100, 10^9]; then runs of length Geom(1/S) (mean S - 1) are
    pre-sorted one after another.  kind: "int" (u32 keys) or "randomBlob30" /
    "zeroBlob30" ((n, 30) u32 records; zeroBlob30 has only the last word
    nonzero); runs of blobs are pre-sorted by their deciding word (the first
    word for randomBlob30 -- ties there are ~n^2 / 2^31 pairs and do not
    matter for an input generator -- the last for zeroBlob30).  Returns
    (data, n)."""
    g = _gen(device, 1000 * seed + S)
    n = int(torch.randint(9 * N // 10, N + 1, (1,), generator=g, device=device).item())
    if kind == "int":
        vals = torch.randint(100, 10 ** 9 + 1, (n,), generator=g, device=device, dtype=torch.int64)
        lead = vals
    elif kind in ("randomBlob30", "zeroBlob30"):
        vals = torch.randint(100, 10 ** 9 + 1, (n, 30), generator=g, device=device, dtype=torch.int64)
        if kind == "zeroBlob30":
            vals[:, :29] = 0
        lead = vals[:, 0] if kind == "randomBlob30" else vals[:, 29]
    else:
        raise ValueError(kind)
    # geometric run lengths with parameter 1/S (support 1, 2, ...)
    p = 1.0 / S
    est = max(16, int(2.5 * n * p) + 64)
    while True:
        u = torch.rand(est, generator=g, device=device, dtype=torch.float64)
        lens = torch.floor(torch.log1p(-u) / math.log1p(-p)).to(torch.int64) + 1 if p < 1 else torch.ones(
            est, dtype=torch.int64, device=device)
        if int(lens.sum()) >= n:
            break
        est *= 2
    cs = torch.cumsum(lens, 0)
    k = int(torch.searchsorted(cs, torch.tensor([n], device=device)).item())
    lens = lens[: k + 1].clone()
    lens[k] -= int(cs[k]) - n
    lens = lens[lens > 0]
    perm = _sort_within_segments(lead, _seg_ids(lens))
    data = vals[perm]
    return _u32_from_i64(data), n


def make(cfg: int, n: int | None = None, seed: int | None = None, device="cpu", **kw):
    f = GENERATORS[cfg]
    args = {}
    if n is not None:
        args["n"] = n
    if seed is not None:
        args["seed"] = seed
    return f(device=device, **args, **kw)


def to_numpy(t: torch.Tensor):
    """Host numpy view of a key/value tensor with the unsigned/f32 dtype."""
    import numpy as np
    t = t.detach().cpu()
    if t.dtype == torch.uint32:
        return t.view(torch.int32).numpy().view(np.uint32)
    if t.dtype == torch.uint64:
        return t.view(torch.int64).numpy().view(np.uint64)
    if t.dtype == torch.float32:
        return t.numpy()
    raise TypeError(t.dtype)


def from_numpy(a, device="cpu") -> torch.Tensor:
    import numpy as np
    if a.dtype == np.uint32:
        return torch.from_numpy(a.view(np.int32).copy()).view(torch.uint32).to(device)
    if a.dtype == np.uint64:
        return torch.from_numpy(a.view(np.int64).copy()).view(torch.uint64).to(device)
    if a.dtype == np.float32:
        return torch.from_numpy(a.copy()).to(device)
    raise TypeError(a.dtype)
