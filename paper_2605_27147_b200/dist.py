"""Multi-GPU sort and merge plan over contiguous shards (BASELINE.json
north_star) -- a thin layer over the library's native protocol
(csrc/comm.cu, declared in include/vmps.h).

One process per GPU.  Rank q holds shard q of the global array (global order
= shard 0, shard 1, ...).  Everything on the method's data path -- the local
sort, the exact splitters (16-ary search over the key order image, counts
summed across ranks), the tie split in rank order, the exchange and the stable
merge of the received pieces, and for the plan the run-detection transfer
tables, their composition and Alg. 1's plan -- runs inside libvmps (kernels
plus the protocol's host arithmetic, NCCL for the collectives).  This module
only marshals: it builds the native communicator from a torch.distributed
process group (rank 0's NCCL unique id is broadcast over the group) and calls

  sort_dist_        vmps_sort_keys_dist / vmps_sort_pairs_dist (in place: rank p
                    keeps global output ranks [off_p, off_p + n_p))
  merge_plan_dist   vmps_merge_plan_dist (this rank's runs and the merges whose
                    boundary lies in its shard; `order` = global execution rank)
  sort_dist_pull    local sort, vmps_dist_cuts (native splitters), CUDA IPC
                    peer mappings of every shard, vmps_merge_pieces reading the
                    co-ranked pieces straight from peer memory

Virtual ranks (tests): ``local_group(g)`` and ``Comm.local`` run the same
native protocol with g threads of one process on one GPU (collectives over
barriers, events and device copies), see tests/test_gpu_comm.py.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import (Comm, LocalGroup, Workspace, dist_cuts, ipc_close, ipc_handle, ipc_open, merge_pieces,
               merge_plan_dist_native, sort_, sort_dist_native_)

_comms: dict = {}


def native_comm(group=None, device: torch.device | None = None) -> Comm:
    """The native NCCL communicator of this rank for a torch.distributed group
    (created once per (group, device) and cached)."""
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = (id(group), dev.index)
    c = _comms.get(key)
    if c is None:
        from . import comm_unique_id
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        c = Comm(rank, world, uid[0], dev.index)
        _comms[key] = c
    return c


def destroy_comms() -> None:
    for c in _comms.values():
        c.destroy()
    _comms.clear()


def local_group(world: int, device: int = 0) -> LocalGroup:
    """An in-process group of `world` virtual ranks on one device."""
    return LocalGroup(world, device)


def sort_dist_(keys: torch.Tensor, vals: torch.Tensor | None = None, group=None, comm: Comm | None = None,
               workspace: Workspace | None = None, scratch: int | None = None, stats: bool = False):
    """Globally stable sort of the concatenation of every rank's shard, in
    place (vmps_sort_*_dist): this rank keeps its element count and ends with
    global output ranks [off, off + n_local)."""
    c = comm if comm is not None else native_comm(group, keys.device)
    return sort_dist_native_(c, keys, vals, scratch=scratch, stats=stats, workspace=workspace)


def merge_plan_dist(keys: torch.Tensor, n_total: int | None = None, group=None, comm: Comm | None = None,
                    workspace: Workspace | None = None):
    """Alg. 1's merge plan of the concatenated shards (vmps_merge_plan_dist):
    this rank's runs (global positions) and the merges whose boundary j lies
    in its shard, with their global execution rank.  n_total: the global n
    (sizes the workspace; gathered over the group when omitted)."""
    c = comm if comm is not None else native_comm(group, keys.device)
    if n_total is None:
        t = torch.tensor([keys.numel()], dtype=torch.int64, device=keys.device)
        dist.all_reduce(t, group=group)
        n_total = int(t.item())
    return merge_plan_dist_native(c, keys, n_total, workspace=workspace)


@dataclass
class DistResult:
    keys: torch.Tensor
    vals: torch.Tensor | None
    send_counts: list[int]
    recv_counts: list[int]
    rounds: int


def sort_dist_pull(keys: torch.Tensor, vals: torch.Tensor | None = None, group=None, comm: Comm | None = None,
                   workspace: Workspace | None = None) -> DistResult:
    """sort_dist with the exchange and the final merge fused:
    after the native splitters every rank maps the other ranks' sorted shards
    (CUDA IPC over NVLink) and merges its co-ranked pieces straight from peer
    memory into its output (vmps_merge_pieces: one TMA-staged 4-way pass for
    g <= 4, two plus a local 2-way pass for g <= 8).  No receive buffer and no
    all-to-all.  Returns this rank's slice [off, off + n_local) as new tensors."""
    c = comm if comm is not None else native_comm(group, keys.device)
    g, me = c.world, c.rank
    dev = keys.device
    sort_(keys, vals, workspace=workspace)
    cut, sizes, rounds = dist_cuts(c, keys, workspace=workspace)
    recv = [cut[q][me + 1] - cut[q][me] for q in range(g)]
    send = [cut[me][p + 1] - cut[me][p] for p in range(g)]
    kb = keys.element_size()
    mine = list(ipc_handle(keys)) + (list(ipc_handle(vals)) if vals is not None else [])
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
        merge_pieces(kp, vp, recv, ok, ov, workspace=workspace)
    torch.cuda.current_stream(dev).synchronize()
    dist.barrier(group=group)  # every peer has read this shard
    for p_, off in opened:
        ipc_close(p_, off)
    return DistResult(ok, ov, send, recv, rounds)
