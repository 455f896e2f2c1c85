"""Multi-GPU sort over contiguous shards (BASELINE.json north_star).

One process per GPU.  Rank q holds shard q of the global array (global order
= shard 0, shard 1, ...).  Steps, all stream-ordered on each rank's device:

  1. local stable sort of the shard            (vmps_sort_keys / vmps_sort_pairs)
  2. exact splitters: for the global output ranks R_t = t N / g, a binary
     search over the key *order image* (u32/f32: 32 bits, u64: 64 bits) finds
     v*_t = the least v with #{x <= v} >= R_t; per-rank counts of "< v" and
     "<= v" come from vmps_count_rank and are summed with an all-reduce.  The
     tie group at v*_t is split in rank order (lower ranks give their equal
     keys first), which is what a stable sort of the concatenation does.
  3. exchange: NCCL all-to-all (torch.distributed.all_to_all_single) of keys
     and payloads; rank p receives the pieces [s_{q,p}, s_{q,p+1}) of every q
  4. local stable merge of the g received pieces in source-rank order
     (vmps_merge_runs, ties to the earlier piece = the lower rank).

Rank p then holds global output ranks [R_p, R_{p+1}).  torch.distributed is the
plumbing (process group, collectives); every step on the data path runs in
libvmps kernels.  The compute ops are passed in as an object so the protocol
itself can be exercised with gloo on CPU (tests/test_dist.py).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import (KEY_F32, KEY_U32, KEY_U64, Workspace, _check, _stream_ptr, key_type, lib,
               sort_)


def image_bits(kt: int) -> int:
    return 64 if kt == KEY_U64 else 32


class VmpsOps:
    """The data-path operations on CUDA tensors, through the C ABI."""

    def __init__(self):
        self.ws = Workspace()

    def local_sort(self, keys, vals):
        sort_(keys, vals, workspace=self.ws)

    def count(self, keys, probes: list[int]) -> tuple[torch.Tensor, torch.Tensor]:
        """(lt, le) int64 device tensors for the probe images."""
        dev = keys.device
        p = torch.tensor([x - (1 << 64) if x >= (1 << 63) else x for x in probes],
                         dtype=torch.int64, device=dev)
        lt = torch.empty(len(probes), dtype=torch.int64, device=dev)
        le = torch.empty(len(probes), dtype=torch.int64, device=dev)
        with torch.cuda.device(dev):
            rc = lib().vmps_count_rank(keys.data_ptr(), keys.numel(), key_type(keys), p.data_ptr(),
                                       len(probes), lt.data_ptr(), le.data_ptr(), _stream_ptr(dev))
        _check(rc, "vmps_count_rank")
        return lt, le

    def merge_runs(self, keys, vals, starts: list[int]):
        n = keys.numel()
        if len(starts) <= 1 or n <= 1:
            return
        kt = key_type(keys)
        L = lib()
        nb = ctypes.c_size_t(0)
        _check(L.vmps_merge_runs_workspace_bytes(n, kt, 1 if vals is not None else 0, len(starts),
                                                 ctypes.byref(nb)), "vmps_merge_runs_workspace_bytes")
        buf = self.ws.get(int(nb.value), keys.device)
        hs = (ctypes.c_uint64 * len(starts))(*starts)
        with torch.cuda.device(keys.device):
            rc = L.vmps_merge_runs(keys.data_ptr(), None if vals is None else vals.data_ptr(), n, kt, hs,
                                   len(starts), buf.data_ptr(), buf.numel(), _stream_ptr(keys.device))
        _check(rc, "vmps_merge_runs")


def _as_int(t: torch.Tensor) -> torch.Tensor:
    """Same-size signed view for collectives (NCCL/gloo have no unsigned types)."""
    if t.dtype in (torch.uint32, torch.float32):
        return t.view(torch.int32)
    if t.dtype == torch.uint64:
        return t.view(torch.int64)
    return t


@dataclass
class DistResult:
    keys: torch.Tensor
    vals: torch.Tensor | None
    splitters: list[int]          # v*_t (order images)
    send_counts: list[int]
    recv_counts: list[int]
    rounds: int


def split_points(R: int, lt_all: list[int], le_all: list[int]) -> list[int]:
    """Per-rank cut s_q for global output rank R, given every rank's counts of
    '< v*' and '<= v*' (v* = least v with sum(le) >= R): all elements < v*,
    then the tie group at v* taken in rank order (stability)."""
    need = R - sum(lt_all)
    cuts = []
    for lt, le in zip(lt_all, le_all):
        eq = le - lt
        take = min(max(need, 0), eq)
        cuts.append(lt + take)
        need -= take
    return cuts


def sort_dist(keys: torch.Tensor, vals: torch.Tensor | None = None, group=None,
              ops=None) -> DistResult:
    """Globally stable sort of the concatenation of every rank's shard.

    Returns this rank's slice [R_p, R_{p+1}) of the global output.
    """
    ops = ops if ops is not None else VmpsOps()
    g = dist.get_world_size(group)
    me = dist.get_rank(group)
    kt = key_type(keys)
    dev = keys.device
    n = keys.numel()
    # 1. local sort
    ops.local_sort(keys, vals)
    # sizes and global ranks
    sz = torch.tensor([n], dtype=torch.int64, device=dev)
    sizes_t = [torch.zeros_like(sz) for _ in range(g)]
    dist.all_gather(sizes_t, sz, group=group)
    sizes = [int(x.item()) for x in sizes_t]
    N = sum(sizes)
    R = [(t * N) // g for t in range(1, g)]
    # 2. splitter search over the order image
    bits = image_bits(kt)
    lo = [0] * (g - 1)
    hi = [(1 << bits) - 1] * (g - 1)
    rounds = 0
    while any(a < b for a, b in zip(lo, hi)):
        mid = [(a + b) // 2 for a, b in zip(lo, hi)]
        _, le = ops.count(keys, mid)
        dist.all_reduce(le, op=dist.ReduceOp.SUM, group=group)
        le_h = le.cpu().tolist()
        for t in range(g - 1):
            if lo[t] < hi[t]:
                if le_h[t] >= R[t]:
                    hi[t] = mid[t]
                else:
                    lo[t] = mid[t] + 1
        rounds += 1
    vstar = lo
    lt, le = ops.count(keys, vstar) if g > 1 else (torch.zeros(0, dtype=torch.int64, device=dev),) * 2
    mine = torch.cat([lt, le]).to(torch.int64)
    allc = [torch.zeros_like(mine) for _ in range(g)]
    dist.all_gather(allc, mine, group=group)
    allc = [c.cpu().tolist() for c in allc]
    # cut[q][t]: elements of rank q that go to ranks < t+1 (t = 0..g-2)
    cut = [[0] * (g + 1) for _ in range(g)]
    for q in range(g):
        cut[q][0] = 0
        cut[q][g] = sizes[q]
    for t in range(g - 1):
        lts = [allc[q][t] for q in range(g)]
        les = [allc[q][g - 1 + t] for q in range(g)]
        pts = split_points(R[t], lts, les)
        for q in range(g):
            cut[q][t + 1] = pts[q]
    send = [cut[me][p + 1] - cut[me][p] for p in range(g)]
    recv = [cut[q][me + 1] - cut[q][me] for q in range(g)]
    # 3. exchange
    out_n = sum(recv)
    ok = torch.empty(out_n, dtype=keys.dtype, device=dev)
    dist.all_to_all_single(_as_int(ok), _as_int(keys), recv, send, group=group)
    ov = None
    if vals is not None:
        ov = torch.empty(out_n, dtype=vals.dtype, device=dev)
        dist.all_to_all_single(_as_int(ov), _as_int(vals), recv, send, group=group)
    # 4. local stable merge of the pieces, in source-rank order
    starts, acc = [], 0
    for c in recv:
        if c > 0:
            starts.append(acc)
        acc += c
    ops.merge_runs(ok, ov, starts)
    return DistResult(ok, ov, vstar, send, recv, rounds)


def sort_dist_(keys: torch.Tensor, vals: torch.Tensor | None = None, group=None) -> DistResult:
    """In-place variant for equal shard sizes (the output slice has the input's length)."""
    res = sort_dist(keys, vals, group)
    if res.keys.numel() != keys.numel():
        raise ValueError("sort_dist_ needs equal shard sizes; use sort_dist")
    keys.copy_(res.keys)
    if vals is not None:
        vals.copy_(res.vals)
    return res
