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

The second protocol, merge_plan_dist, computes Alg. 1's merge plan of the
concatenated shards without moving keys (see the section comment below).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import (KEY_U64, Workspace, _check, _stream_ptr, key_type, lib,
               minrun_for, sort_)


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


def _cuts(keys, vals, group, ops):
    """Steps 1-2: local sort and exact splitters.  Returns (cut, sizes,
    splitters, rounds) with cut[q][t] = elements of rank q that go to ranks < t."""
    g = dist.get_world_size(group)
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
    return cut, sizes, vstar, rounds


def sort_dist(keys: torch.Tensor, vals: torch.Tensor | None = None, group=None,
              ops=None) -> DistResult:
    """Globally stable sort of the concatenation of every rank's shard.

    Returns this rank's slice [R_p, R_{p+1}) of the global output.
    """
    ops = ops if ops is not None else VmpsOps()
    g = dist.get_world_size(group)
    me = dist.get_rank(group)
    dev = keys.device
    cut, sizes, vstar, rounds = _cuts(keys, vals, group, ops)
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


# ---------------------------------------------------------------------------
# Distributed merge plan: Alg. 1's plan of the
# concatenation of the ranks' shards, without moving the keys.
#
# Run detection is a left-to-right chain (ExtractRun, P:399 / P:756): each
# shard computes its transfer table (chain state at its start -> state at its
# end, runs started) with vmps_shard_chain; composing the g tables from
# START(0) on the host gives every shard its entry state and run count; each
# shard then emits its run starts (global positions) with vmps_shard_runs.
# The run list is assembled on every rank and vmps_plan_from_runs computes
# powers, tree and Alg. 1's order (Alg. 1) -- a replicated,
# O(r)-sized step.  Inputs crossing the shard edges: the previous shard's last
# key (descent bit at the shard start) and the next HALO keys of the global
# array (runs that cross the shard end are classified exactly).
# ---------------------------------------------------------------------------

ST_END = 255


def halo_len(minrun: int) -> int:
    """Keys after a shard's end its run classification may read: minrun + 8."""
    return minrun + 8


def compose_tables(tables: list) -> tuple[list[int], list[int]]:
    """Entry states and run counts of consecutive shards from START(0).
    tables[q]: the shard's transfer table (a list of 64-bit values: exit state
    << 32 | runs started, indexed by entry state), or None for an empty shard
    (identity, no runs)."""
    st = 0
    entries, counts = [], []
    for t in tables:
        entries.append(st)
        if t is None or st == ST_END:
            counts.append(0)
            continue
        v = int(t[st]) & 0xFFFFFFFFFFFFFFFF
        counts.append(v & 0xFFFFFFFF)
        st = v >> 32
    return entries, counts


def halo_from_heads(me: int, heads: list, sizes: list[int], need: int):
    """The first `need` keys after shard `me` (fewer at the global end), from
    the other shards' heads (heads[p] = shard p's first min(need, n_p) keys)."""
    parts, got = [], 0
    for p in range(me + 1, len(sizes)):
        if got >= need:
            break
        take = min(sizes[p], need - got, len(heads[p]))
        if take > 0:
            parts.append(heads[p][:take])
            got += take
    return parts


def prev_owner(me: int, sizes: list[int]) -> int:
    """The nearest non-empty shard before `me` (-1 if none)."""
    for p in range(me - 1, -1, -1):
        if sizes[p] > 0:
            return p
    return -1


class PlanOps:
    """The data-path operations of the distributed plan, through the C ABI."""

    def __init__(self):
        self.ws = Workspace()

    def chain(self, keys, minrun, n_end, prev, halo):
        from . import shard_chain
        return shard_chain(keys, minrun, n_end, prev, halo, workspace=self.ws)

    def runs(self, keys, minrun, n_end, prev, halo, entry, count, offset, out_starts):
        from . import shard_runs
        return shard_runs(keys, minrun, n_end, entry, count, offset, prev, halo, out=out_starts,
                          workspace=self.ws)[1]

    def plan(self, starts, n):
        from . import plan_from_runs
        return plan_from_runs(starts, n, workspace=self.ws)


@dataclass
class DistPlan:
    run_start: torch.Tensor     # int64 (r,), global positions
    run_kind: torch.Tensor      # uint8 (r,)
    merges: torch.Tensor        # int64 (r - 1, 4): (i, j, k, power), Alg. 1's order
    minrun: int
    entries: list[int]          # chain state at each shard's start
    counts: list[int]           # runs starting in each shard


def _cat(parts):
    if not parts:
        return None
    return torch.cat(parts).contiguous() if len(parts) > 1 else parts[0].contiguous()


def merge_plan_shards(shards: list[torch.Tensor], ops=None) -> DistPlan:
    """The same protocol for g shards held by one process (virtual ranks):
    the plan of torch.cat(shards), each shard processed on its own."""
    ops = ops if ops is not None else PlanOps()
    sizes = [s.numel() for s in shards]
    N = sum(sizes)
    if N == 0:
        raise ValueError("empty array")
    dev = next(s.device for s in shards if s.numel() > 0)
    minrun = minrun_for(N)
    H = halo_len(minrun)
    offs = [sum(sizes[:q]) for q in range(len(shards))]
    heads = [s[:min(H, s.numel())] for s in shards]
    tables = []
    for q, s in enumerate(shards):
        if sizes[q] == 0:
            tables.append(None)
            continue
        pq = prev_owner(q, sizes)
        prev = shards[pq][-1:].contiguous() if pq >= 0 else None
        halo = _cat(halo_from_heads(q, heads, sizes, H))
        tables.append(ops.chain(s, minrun, N - offs[q], prev, halo).cpu().tolist())
    entries, counts = compose_tables(tables)
    r = sum(counts)
    starts = torch.empty(r + 1, dtype=torch.int64, device=dev)
    kinds = torch.empty(r, dtype=torch.uint8, device=dev)
    o = 0
    for q, s in enumerate(shards):
        if counts[q] == 0:
            continue
        pq = prev_owner(q, sizes)
        prev = shards[pq][-1:].contiguous() if pq >= 0 else None
        halo = _cat(halo_from_heads(q, heads, sizes, H))
        k = ops.runs(s, minrun, N - offs[q], prev, halo, entries[q], counts[q], offs[q], starts[o:o + counts[q]])
        kinds[o:o + counts[q]].copy_(k)
        o += counts[q]
    starts[r] = N
    merges = ops.plan(starts, N)
    return DistPlan(starts[:r], kinds, merges, minrun, entries, counts)


def merge_plan_dist(keys: torch.Tensor, group=None, ops=None) -> DistPlan:
    """Alg. 1's merge plan of the concatenation of every rank's shard (global
    order = rank order), replicated on every rank; the keys do not move."""
    ops = ops if ops is not None else PlanOps()
    g = dist.get_world_size(group)
    me = dist.get_rank(group)
    dev = keys.device
    n = keys.numel()
    sz = torch.tensor([n], dtype=torch.int64, device=dev)
    sizes_t = [torch.zeros_like(sz) for _ in range(g)]
    dist.all_gather(sizes_t, sz, group=group)
    sizes = [int(x.item()) for x in sizes_t]
    N = sum(sizes)
    if N == 0:
        raise ValueError("empty array")
    off = sum(sizes[:me])
    minrun = minrun_for(N)
    H = halo_len(minrun)
    # edge keys: every shard's head (first H keys, padded) and last key
    edge = torch.zeros(H + 1, dtype=keys.dtype, device=dev)
    h = min(H, n)
    if h:
        edge[:h].copy_(keys[:h])
        edge[H:].copy_(keys[n - 1:])
    edges = [torch.empty_like(edge) for _ in range(g)]
    dist.all_gather([_as_int(e) for e in edges], _as_int(edge), group=group)
    heads = [e[:min(H, sizes[p])] for p, e in enumerate(edges)]
    pq = prev_owner(me, sizes)
    prev = edges[pq][H:].contiguous() if pq >= 0 else None
    halo = _cat(halo_from_heads(me, heads, sizes, H))
    # transfer tables -> entry states and run counts (host composition)
    mine = ops.chain(keys, minrun, N - off, prev, halo) if n else torch.zeros(3 * minrun, dtype=torch.int64,
                                                                            device=dev)
    tabs = [torch.empty_like(mine) for _ in range(g)]
    dist.all_gather(tabs, mine, group=group)
    tables = [t.cpu().tolist() if sizes[p] else None for p, t in enumerate(tabs)]
    entries, counts = compose_tables(tables)
    r = sum(counts)
    o = sum(counts[:me])
    starts = torch.empty(r + 1, dtype=torch.int64, device=dev)
    kinds = torch.empty(max(r, 1), dtype=torch.uint8, device=dev)
    if counts[me]:
        k = ops.runs(keys, minrun, N - off, prev, halo, entries[me], counts[me], off, starts[o:o + counts[me]])
        kinds[o:o + counts[me]].copy_(k)
    # every rank's run list to every rank (in place, rank order)
    a = 0
    for p in range(g):
        if counts[p]:
            dist.broadcast(starts[a:a + counts[p]], src=p, group=group)
            dist.broadcast(kinds[a:a + counts[p]], src=p, group=group)
        a += counts[p]
    starts[r] = N
    merges = ops.plan(starts, N)
    return DistPlan(starts[:r], kinds[:r], merges, minrun, entries, counts)



def sort_dist_pull(keys: torch.Tensor, vals: torch.Tensor | None = None, group=None,
                   ops=None) -> DistResult:
    """sort_dist with the exchange and the final merge fused:
    after the splitters, every rank maps the other ranks' sorted shards
    (CUDA IPC over NVLink; vmps_ipc_handle / vmps_ipc_open) and merges its
    co-ranked pieces straight from peer memory into its output
    (vmps_merge_pieces: one TMA-staged 4-way pass for g <= 4, two plus a
    local 2-way pass for g <= 8).  No receive buffer, no all-to-all: one HBM
    write + read of the shard fewer than all-to-all + merge.  Barriers keep a
    shard alive until every peer has read it."""
    from . import ipc_close, ipc_handle, ipc_open, merge_pieces
    ops = ops if ops is not None else VmpsOps()
    g = dist.get_world_size(group)
    me = dist.get_rank(group)
    dev = keys.device
    cut, sizes, vstar, rounds = _cuts(keys, vals, group, ops)
    recv = [cut[q][me + 1] - cut[q][me] for q in range(g)]
    send = [cut[me][p + 1] - cut[me][p] for p in range(g)]
    kb = keys.element_size()
    # peer mappings of every shard (keys, values)
    hk, ok_ = ipc_handle(keys)
    mine = [hk, ok_]
    if vals is not None:
        hv, ov_ = ipc_handle(vals)
        mine += [hv, ov_]
    allh = [None] * g
    dist.all_gather_object(allh, mine, group=group)
    kptr, vptr, opened = [], [], []
    for q in range(g):
        if q == me:
            kptr.append(keys.data_ptr())
            vptr.append(vals.data_ptr() if vals is not None else 0)
            continue
        pk = ipc_open(allh[q][0], allh[q][1])
        opened.append((pk, allh[q][1]))
        kptr.append(pk)
        if vals is not None:
            pv = ipc_open(allh[q][2], allh[q][3])
            opened.append((pv, allh[q][3]))
            vptr.append(pv)
    torch.cuda.current_stream(dev).synchronize()
    dist.barrier(group=group)  # every shard is sorted and mapped
    out_n = sum(recv)
    ok = torch.empty(out_n, dtype=keys.dtype, device=dev)
    ov = torch.empty(out_n, dtype=vals.dtype, device=dev) if vals is not None else None
    kp = [kptr[q] + cut[q][me] * kb for q in range(g)]
    vp = [vptr[q] + cut[q][me] * 4 for q in range(g)] if vals is not None else None
    if out_n:
        merge_pieces(kp, vp, recv, ok, ov)
    torch.cuda.current_stream(dev).synchronize()
    dist.barrier(group=group)  # every peer has read this shard
    for p_, off in opened:
        ipc_close(p_, off)
    return DistResult(ok, ov, vstar, send, recv, rounds)
