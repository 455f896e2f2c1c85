"""B200-native (sm_100a) Virtual-Memory Powersort hot path -- Python binding.

Thin ctypes marshalling over ``libvmps.so`` (C ABI in ``include/vmps.h``):
torch supplies device memory, the current CUDA stream and (for the
multi-GPU path) process groups; every step of the sort runs in the library's
CUDA kernels.  There is no CPU fallback: importing works anywhere, but any
call raises if ``libvmps.so`` is missing or no CUDA device is present.

Names follow include/vmps.h: ``sort_`` (vmps_sort_keys / vmps_sort_pairs),
``merge_plan`` (vmps_merge_plan), ``workspace_bytes``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VMPS_LIB") or os.path.join(_HERE, "libvmps.so")

KEY_U32, KEY_U64, KEY_F32 = 0, 1, 2
OK, ERR_INVALID_ARG, ERR_ALLOC, ERR_BUDGET, ERR_CUDA, ERR_NCCL, ERR_INTERNAL = range(7)
SCRATCH_UNBOUNDED = -1
RUN_ASC, RUN_DESC, RUN_EXT = 0, 1, 2

_STATUS = {0: "ok", 1: "invalid argument", 2: "allocation failed", 3: "budget too small",
           4: "CUDA error", 5: "NCCL error", 6: "internal error"}


class VmpsError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        super().__init__(f"{where}: {_STATUS.get(status, status)}" + (f" ({detail})" if detail else ""))


class Stats(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("runs", ctypes.c_uint64), ("merges", ctypes.c_uint64),
                ("merge_cost_M", ctypes.c_uint64), ("fused_M", ctypes.c_uint64),
                ("reversed_elems", ctypes.c_uint64), ("extended_runs", ctypes.c_uint64),
                ("max_power", ctypes.c_uint32), ("levels_executed", ctypes.c_uint32),
                ("minrun", ctypes.c_uint32), ("block_elems", ctypes.c_uint32),
                ("rounds", ctypes.c_uint64), ("peak_extra_device_bytes", ctypes.c_uint64),
                ("scratch_bytes", ctypes.c_uint64), ("metadata_bytes", ctypes.c_uint64),
                ("hbm_merge_elems", ctypes.c_uint64)]

    def as_dict(self) -> dict:
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


class MergeRec(ctypes.Structure):
    _fields_ = [("i", ctypes.c_uint64), ("j", ctypes.c_uint64), ("k", ctypes.c_uint64),
                ("power", ctypes.c_uint32), ("order", ctypes.c_uint32)]


EXPORTS = ("vmps_workspace_bytes", "vmps_sort_keys", "vmps_sort_pairs", "vmps_merge_plan",
           "vmps_count_rank", "vmps_merge_runs_workspace_bytes", "vmps_merge_runs",
           "vmps_status_string", "vmps_last_error", "vmps_profile_enable", "vmps_profile_read",
           "vmps_test_set_minrun", "vmps_test_set_tiles", "vmps_test_set_mode",
           "vmps_test_set_leaf", "vmps_sort_keys_host", "vmps_sort_pairs_host",
           "vmps_shard_workspace_bytes", "vmps_shard_chain", "vmps_shard_runs", "vmps_plan_workspace_bytes",
           "vmps_plan_from_runs", "vmps_comm_unique_id", "vmps_comm_init", "vmps_comm_destroy",
           "vmps_comm_last_error", "vmps_dist_workspace_bytes", "vmps_sort_keys_dist", "vmps_sort_pairs_dist",
           "vmps_merge_plan_dist_workspace_bytes", "vmps_merge_plan_dist", "vmps_sort_records_workspace_bytes",
           "vmps_sort_records", "vmps_records_last_error", "vmps_merge_pieces_workspace_bytes",
           "vmps_merge_pieces", "vmps_ipc_handle", "vmps_ipc_open", "vmps_ipc_close",
           "vmps_local_group_create", "vmps_local_group_destroy", "vmps_comm_init_local",
           "vmps_dist_cuts_workspace_bytes", "vmps_dist_cuts", "vmps_splitter_probes", "vmps_splitter_update",
           "vmps_split_points", "vmps_compose_tables", "vmps_merge_plan_dist_capacity", "vmps_test_set_bd_chunk",
           "vmps_merge_runs_bounded_workspace_bytes", "vmps_merge_runs_bounded")

_lib = None


def lib() -> ctypes.CDLL:
    """Load libvmps.so (built in-tree by ``build.py``); raise loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2605_27147_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, u64, i64, sz = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_size_t
        L.vmps_workspace_bytes.argtypes = [u64, ctypes.c_int, ctypes.c_int, i64, ctypes.POINTER(sz)]
        L.vmps_sort_keys.argtypes = [vp, u64, ctypes.c_int, i64, vp, sz, vp, ctypes.POINTER(Stats)]
        L.vmps_sort_pairs.argtypes = [vp, vp, u64, ctypes.c_int, i64, vp, sz, vp, ctypes.POINTER(Stats)]
        L.vmps_sort_keys_host.argtypes = [vp, vp, u64, ctypes.c_int, i64, vp, vp, sz, vp, ctypes.POINTER(Stats)]
        L.vmps_sort_pairs_host.argtypes = [vp, vp, vp, vp, u64, ctypes.c_int, i64, vp, vp, vp, sz, vp,
                                           ctypes.POINTER(Stats)]
        u32, ci = ctypes.c_uint32, ctypes.c_int
        L.vmps_shard_workspace_bytes.argtypes = [u64, ci, u32, ctypes.POINTER(sz)]
        L.vmps_shard_chain.argtypes = [vp, u64, ci, u32, u32, vp, vp, u32, vp, vp, sz, vp]
        L.vmps_shard_runs.argtypes = [vp, u64, ci, u32, u32, vp, vp, u32, u32, u64, u64, vp, vp, vp, sz, vp]
        L.vmps_plan_workspace_bytes.argtypes = [u64, ctypes.POINTER(sz)]
        L.vmps_plan_from_runs.argtypes = [vp, u64, u64, vp, vp, sz, vp]
        for f in ("vmps_shard_workspace_bytes", "vmps_shard_chain", "vmps_shard_runs", "vmps_plan_workspace_bytes",
                  "vmps_plan_from_runs"):
            getattr(L, f).restype = ctypes.c_int
        i64 = ctypes.c_int64
        L.vmps_comm_unique_id.argtypes = [vp]
        L.vmps_comm_init.argtypes = [ctypes.POINTER(vp), ci, ci, vp, ci]
        L.vmps_comm_destroy.argtypes = [vp]
        L.vmps_comm_last_error.restype = ctypes.c_char_p
        L.vmps_dist_workspace_bytes.argtypes = [u64, ci, ci, ci, i64, ctypes.POINTER(sz)]
        L.vmps_sort_keys_dist.argtypes = [vp, vp, u64, ci, i64, vp, sz, vp, vp]
        L.vmps_sort_pairs_dist.argtypes = [vp, vp, vp, u64, ci, i64, vp, sz, vp, vp]
        L.vmps_merge_plan_dist_workspace_bytes.argtypes = [u64, u64, ci, ci, ctypes.POINTER(sz)]
        L.vmps_merge_plan_dist_capacity.argtypes = [u64, u64, ctypes.POINTER(u64)]
        L.vmps_merge_plan_dist_capacity.restype = ctypes.c_int
        L.vmps_merge_plan_dist.argtypes = [vp, vp, u64, ci, vp, vp, vp, u64, ctypes.POINTER(u64),
                                           ctypes.POINTER(u64), vp, sz, vp]
        L.vmps_merge_pieces_workspace_bytes.argtypes = [u64, ci, ci, u32, ctypes.POINTER(sz)]
        L.vmps_merge_pieces.argtypes = [vp, vp, vp, u32, vp, vp, ci, vp, sz, vp]
        L.vmps_ipc_handle.argtypes = [vp, vp, ctypes.POINTER(u64)]
        L.vmps_ipc_open.argtypes = [vp, u64, ctypes.POINTER(vp)]
        L.vmps_ipc_close.argtypes = [vp, u64]
        for f in ("vmps_merge_pieces_workspace_bytes", "vmps_merge_pieces", "vmps_ipc_handle", "vmps_ipc_open",
                  "vmps_ipc_close"):
            getattr(L, f).restype = ctypes.c_int
        L.vmps_local_group_create.argtypes = [ci, ci, ctypes.POINTER(vp)]
        L.vmps_local_group_destroy.argtypes = [vp]
        L.vmps_comm_init_local.argtypes = [ctypes.POINTER(vp), ci, vp, ci]
        L.vmps_dist_cuts_workspace_bytes.argtypes = [ci, ctypes.POINTER(sz)]
        L.vmps_dist_cuts.argtypes = [vp, vp, u64, ci, vp, vp, vp, vp, sz, vp]
        L.vmps_splitter_probes.argtypes = [u32, vp, vp, vp, vp, ctypes.POINTER(u32)]
        L.vmps_splitter_update.argtypes = [u32, vp, vp, vp, vp, vp, vp]
        L.vmps_split_points.argtypes = [u32, u64, vp, vp, vp]
        L.vmps_compose_tables.argtypes = [u32, u32, vp, vp, vp, vp]
        for f in ("vmps_local_group_create", "vmps_local_group_destroy", "vmps_comm_init_local",
                  "vmps_dist_cuts_workspace_bytes", "vmps_dist_cuts", "vmps_splitter_probes",
                  "vmps_splitter_update", "vmps_split_points", "vmps_compose_tables"):
            getattr(L, f).restype = ctypes.c_int
        L.vmps_sort_records_workspace_bytes.argtypes = [u64, u32, ctypes.POINTER(sz)]
        L.vmps_sort_records.argtypes = [vp, vp, vp, u64, u32, vp, sz, vp]
        L.vmps_records_last_error.restype = ctypes.c_char_p
        for f in ("vmps_sort_records_workspace_bytes", "vmps_sort_records"):
            getattr(L, f).restype = ctypes.c_int
        for f in ("vmps_comm_unique_id", "vmps_comm_init", "vmps_comm_destroy", "vmps_dist_workspace_bytes",
                  "vmps_sort_keys_dist", "vmps_sort_pairs_dist", "vmps_merge_plan_dist_workspace_bytes",
                  "vmps_merge_plan_dist"):
            getattr(L, f).restype = ctypes.c_int
        L.vmps_merge_plan.argtypes = [vp, u64, ctypes.c_int, vp, vp, vp, u64, ctypes.POINTER(u64),
                                      vp, sz, vp]
        L.vmps_count_rank.argtypes = [vp, u64, ctypes.c_int, vp, ctypes.c_uint32, vp, vp, vp]
        L.vmps_merge_runs_workspace_bytes.argtypes = [u64, ctypes.c_int, ctypes.c_int, ctypes.c_uint32,
                                                      ctypes.POINTER(sz)]
        L.vmps_merge_runs.argtypes = [vp, vp, u64, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64),
                                      ctypes.c_uint32, vp, sz, vp]
        for f in ("vmps_workspace_bytes", "vmps_sort_keys", "vmps_sort_pairs", "vmps_sort_keys_host",
                  "vmps_sort_pairs_host", "vmps_merge_plan",
                  "vmps_count_rank", "vmps_merge_runs_workspace_bytes", "vmps_merge_runs"):
            getattr(L, f).restype = ctypes.c_int
        L.vmps_status_string.restype = ctypes.c_char_p
        L.vmps_status_string.argtypes = [ctypes.c_int]
        L.vmps_last_error.restype = ctypes.c_char_p
        L.vmps_last_error.argtypes = []
        L.vmps_profile_enable.argtypes = [ctypes.c_int]
        L.vmps_profile_enable.restype = None
        L.vmps_profile_read.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                                        ctypes.POINTER(u64), ctypes.POINTER(u64)]
        L.vmps_profile_read.restype = ctypes.c_int
        L.vmps_test_set_minrun.argtypes = [ctypes.c_uint32]
        L.vmps_test_set_minrun.restype = None
        L.vmps_test_set_mode.argtypes = [ctypes.c_int]
        L.vmps_test_set_mode.restype = None
        L.vmps_test_set_leaf.argtypes = [ctypes.c_int]
        L.vmps_test_set_leaf.restype = None
        L.vmps_test_set_tiles.argtypes = [ctypes.c_uint32] * 3
        L.vmps_test_set_tiles.restype = None
        L.vmps_merge_runs_bounded_workspace_bytes.argtypes = [u64, ci, ci, u32, i64, ctypes.POINTER(sz)]
        L.vmps_merge_runs_bounded.argtypes = [vp, vp, u64, ci, ctypes.POINTER(u64), u32, i64, vp, sz, vp]
        L.vmps_merge_runs_bounded_workspace_bytes.restype = ctypes.c_int
        L.vmps_merge_runs_bounded.restype = ctypes.c_int
        L.vmps_test_set_bd_chunk.argtypes = [ctypes.c_uint32]
        L.vmps_test_set_bd_chunk.restype = None
        _lib = L
    return _lib


def _check(rc: int, where: str):
    if rc != 0:
        raise VmpsError(rc, where, lib().vmps_last_error().decode())


def key_type(t: torch.Tensor) -> int:
    if t.dtype in (torch.uint32, torch.int32):
        return KEY_U32
    if t.dtype in (torch.uint64, torch.int64):
        return KEY_U64
    if t.dtype == torch.float32:
        return KEY_F32
    raise TypeError(f"unsupported key dtype {t.dtype} (u32/u64/f32; int32/int64 are read as unsigned)")


def workspace_bytes(n: int, kt: int, has_vals: int, scratch: int = SCRATCH_UNBOUNDED) -> int:
    out = ctypes.c_size_t(0)
    _check(lib().vmps_workspace_bytes(n, kt, has_vals, scratch, ctypes.byref(out)),
           "vmps_workspace_bytes")
    return int(out.value)


class Workspace:
    """A reusable device workspace (grown on demand) for repeated sorts.

    The C ABI requires concurrent calls to use separate workspaces; one
    Workspace may still be used from several streams one after another: every
    use on a stream other than the allocating one is recorded
    (``record_stream``), so the caching allocator does not hand the memory
    out again while that stream's sort may still read it (also when the
    buffer is replaced by a larger one)."""

    def __init__(self, device=None):
        self.device = torch.device(device) if device is not None else None
        self.buf = None
        self._alloc_stream = None

    def get(self, nbytes: int, device, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        device = torch.device(device)
        cur = stream if stream is not None else torch.cuda.current_stream(device)
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = None
            with torch.cuda.stream(cur):
                self.buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
            self._alloc_stream = cur.cuda_stream
        elif cur.cuda_stream != self._alloc_stream:
            self.buf.record_stream(cur)
        return self.buf


# default workspaces, one per (device, stream, thread): sorts on different
# streams never share one implicitly, nor do threads that torch hands the same
# pooled stream
_default_ws: dict = {}


def _default_workspace(device, stream: torch.cuda.Stream | None = None) -> Workspace:
    import threading
    device = torch.device(device)
    sp = (stream if stream is not None else torch.cuda.current_stream(device)).cuda_stream
    return _default_ws.setdefault((device, sp, threading.get_ident()), Workspace())


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def sort_(keys: torch.Tensor, values: torch.Tensor | None = None, scratch: int | None = None,
          stats: bool = False, workspace: Workspace | None = None):
    """Stable in-place sort of a contiguous CUDA tensor of u32/u64/f32 keys
    (optionally permuting a u32/int32 payload) on the current stream.
    Returns a stats dict when ``stats`` (synchronises), else None."""
    if not keys.is_cuda:
        raise ValueError("keys must be a CUDA tensor (no CPU fallback)")
    if not keys.is_contiguous() or keys.dim() != 1:
        raise ValueError("keys must be a contiguous 1-D tensor")
    kt = key_type(keys)
    n = keys.numel()
    if values is not None:
        if values.dtype not in (torch.uint32, torch.int32) or values.numel() != n:
            raise ValueError("values must be u32/int32 with the same length as keys")
        if not values.is_contiguous() or values.device != keys.device:
            raise ValueError("values must be contiguous on the keys' device")
    sc = SCRATCH_UNBOUNDED if scratch is None else int(scratch)
    nbytes = workspace_bytes(n, kt, 1 if values is not None else 0, sc)
    ws = workspace if workspace is not None else _default_workspace(keys.device)
    buf = ws.get(nbytes, keys.device)
    st = Stats()
    sp = ctypes.byref(st) if stats else None
    L = lib()
    with torch.cuda.device(keys.device):
        s = _stream_ptr(keys.device)
        if values is None:
            rc = L.vmps_sort_keys(keys.data_ptr(), n, kt, sc, buf.data_ptr(), buf.numel(), s, sp)
            _check(rc, "vmps_sort_keys")
        else:
            rc = L.vmps_sort_pairs(keys.data_ptr(), values.data_ptr(), n, kt, sc, buf.data_ptr(),
                                   buf.numel(), s, sp)
            _check(rc, "vmps_sort_pairs")
    return st.as_dict() if stats else None


def sort_host_(keys: torch.Tensor, values: torch.Tensor | None = None, scratch: int | None = None,
               device=None, out_keys: torch.Tensor | None = None, out_values: torch.Tensor | None = None,
               d_keys: torch.Tensor | None = None, d_values: torch.Tensor | None = None,
               workspace: Workspace | None = None, stream: torch.cuda.Stream | None = None) -> None:
    """End-to-end stable sort of HOST tensors (pinned for overlap) through
    vmps_sort_*_host: copy in, device sort, copy back into ``out_keys`` /
    ``out_values`` (default: in place), all enqueued on ``stream`` (default:
    the current stream of ``device``).  Device buffers are allocated unless
    given.  Returns after enqueueing; the output holds the result once the
    stream completes."""
    def _host(t, name):
        if t is None:
            return
        if t.is_cuda or t.dim() != 1 or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous 1-D host tensor")
    _host(keys, "keys"); _host(values, "values"); _host(out_keys, "out_keys"); _host(out_values, "out_values")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    kt = key_type(keys)
    n = keys.numel()
    if values is not None and (values.numel() != n or values.dtype not in (torch.uint32, torch.int32)):
        raise ValueError("values must be u32/int32 with the keys' length")
    if out_keys is not None and (out_keys.numel() != n or out_keys.element_size() != keys.element_size()):
        raise ValueError("out_keys must match keys")
    if out_values is not None and (values is None or out_values.numel() != n or out_values.element_size() != 4):
        raise ValueError("out_values must match values")
    dk = d_keys if d_keys is not None else torch.empty_like(keys, device=dev)
    dv = None
    if values is not None:
        dv = d_values if d_values is not None else torch.empty_like(values, device=dev)
    if stream is not None:  # buffers allocated here are used on `stream`
        if d_keys is None:
            dk.record_stream(stream)
        if dv is not None and d_values is None:
            dv.record_stream(stream)
    sc = SCRATCH_UNBOUNDED if scratch is None else int(scratch)
    nbytes = workspace_bytes(n, kt, 1 if values is not None else 0, sc)
    ws = workspace if workspace is not None else _default_workspace(dev, stream)
    buf = ws.get(nbytes, dev, stream)
    L = lib()
    ko = out_keys.data_ptr() if out_keys is not None else None
    with torch.cuda.device(dev):
        s = stream.cuda_stream if stream is not None else _stream_ptr(dev)
        if values is None:
            rc = L.vmps_sort_keys_host(keys.data_ptr(), ko, n, kt, sc, dk.data_ptr(), buf.data_ptr(), buf.numel(),
                                       s, None)
            _check(rc, "vmps_sort_keys_host")
        else:
            vo = out_values.data_ptr() if out_values is not None else None
            rc = L.vmps_sort_pairs_host(keys.data_ptr(), values.data_ptr(), ko, vo, n, kt, sc, dk.data_ptr(),
                                        dv.data_ptr(), buf.data_ptr(), buf.numel(), s, None)
            _check(rc, "vmps_sort_pairs_host")


@dataclass
class Plan:
    run_start: torch.Tensor  # int64 [r] (device)
    run_kind: torch.Tensor   # uint8 [r] (device), RUN_* bits
    merges: torch.Tensor     # int64 [r-1, 4] (i, j, k, power) in Alg. 1's execution order


def merge_plan(keys: torch.Tensor, workspace: Workspace | None = None) -> Plan:
    """Alg. 1's merge plan of a CUDA key tensor (keys are only read)."""
    if not keys.is_cuda or not keys.is_contiguous() or keys.dim() != 1:
        raise ValueError("keys must be a contiguous 1-D CUDA tensor")
    kt = key_type(keys)
    n = keys.numel()
    dev = keys.device
    nbytes = workspace_bytes(n, kt, -1)
    ws = workspace if workspace is not None else _default_workspace(dev)
    buf = ws.get(nbytes, dev)
    L = lib()
    nr = ctypes.c_uint64(0)
    cap = max(n, 1)
    # run count bound: n // minrun + 2 (minrun from the paper's rule or the test hook)
    rs = torch.empty(cap + 1, dtype=torch.int64, device=dev)
    rk = torch.empty(cap + 1, dtype=torch.uint8, device=dev)
    mg = torch.empty((cap + 1) * 4, dtype=torch.int64, device=dev)  # 32-byte records
    with torch.cuda.device(dev):
        rc = L.vmps_merge_plan(keys.data_ptr(), n, kt, rs.data_ptr(), rk.data_ptr(), mg.data_ptr(),
                               cap, ctypes.byref(nr), buf.data_ptr(), buf.numel(), _stream_ptr(dev))
        _check(rc, "vmps_merge_plan")
    r = int(nr.value)
    recs = mg[: 4 * max(r - 1, 0)].view(-1, 4)
    power = (recs[:, 3] & 0xFFFFFFFF)
    merges = torch.stack([recs[:, 0], recs[:, 1], recs[:, 2], power], dim=1)
    return Plan(rs[:r], rk[:r], merges)


def shard_chain(keys: torch.Tensor, minrun: int, n_end: int, prev: torch.Tensor | None = None,
                halo: torch.Tensor | None = None, workspace: Workspace | None = None) -> torch.Tensor:
    """vmps_shard_chain: the shard's run-detection transfer table, 3 minrun
    int64 values (exit state << 32 | runs started) on the keys' device."""
    kt = key_type(keys)
    dev = keys.device
    L = lib()
    nb = ctypes.c_size_t(0)
    _check(L.vmps_shard_workspace_bytes(keys.numel(), kt, minrun, ctypes.byref(nb)), "vmps_shard_workspace_bytes")
    ws = workspace if workspace is not None else _default_workspace(dev)
    buf = ws.get(int(nb.value), dev)
    tab = torch.empty(3 * minrun, dtype=torch.int64, device=dev)
    nh = 0 if halo is None else halo.numel()
    with torch.cuda.device(dev):
        rc = L.vmps_shard_chain(keys.data_ptr(), keys.numel(), kt, minrun, min(n_end, 0xFFFFFFFF),
                                None if prev is None else prev.data_ptr(), None if nh == 0 else halo.data_ptr(),
                                nh, tab.data_ptr(), buf.data_ptr(), buf.numel(), _stream_ptr(dev))
    _check(rc, "vmps_shard_chain")
    return tab


def shard_runs(keys: torch.Tensor, minrun: int, n_end: int, entry_state: int, count: int, offset: int,
               prev: torch.Tensor | None = None, halo: torch.Tensor | None = None, out: torch.Tensor | None = None,
               workspace: Workspace | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """vmps_shard_runs: the shard's `count` run starts (global int64 positions,
    written into `out` if given) and run kinds (uint8)."""
    kt = key_type(keys)
    dev = keys.device
    L = lib()
    nb = ctypes.c_size_t(0)
    _check(L.vmps_shard_workspace_bytes(keys.numel(), kt, minrun, ctypes.byref(nb)), "vmps_shard_workspace_bytes")
    ws = workspace if workspace is not None else _default_workspace(dev)
    buf = ws.get(int(nb.value), dev)
    rs = out if out is not None else torch.empty(max(count, 1), dtype=torch.int64, device=dev)
    rk = torch.empty(max(count, 1), dtype=torch.uint8, device=dev)
    nh = 0 if halo is None else halo.numel()
    with torch.cuda.device(dev):
        rc = L.vmps_shard_runs(keys.data_ptr(), keys.numel(), kt, minrun, min(n_end, 0xFFFFFFFF),
                               None if prev is None else prev.data_ptr(), None if nh == 0 else halo.data_ptr(),
                               nh, entry_state, count, offset, rs.data_ptr(), rk.data_ptr(), buf.data_ptr(),
                               buf.numel(), _stream_ptr(dev))
    _check(rc, "vmps_shard_runs")
    return rs[:count], rk[:count]


def plan_from_runs(run_start: torch.Tensor, n: int, workspace: Workspace | None = None) -> torch.Tensor:
    """vmps_plan_from_runs: Alg. 1's merge records (r - 1, 4) = (i, j, k, power)
    for the r runs whose int64 starts are run_start[0..r) and run_start[r] = n."""
    r = run_start.numel() - 1
    dev = run_start.device
    if r < 2:
        return torch.empty((0, 4), dtype=torch.int64, device=dev)
    L = lib()
    nb = ctypes.c_size_t(0)
    _check(L.vmps_plan_workspace_bytes(r, ctypes.byref(nb)), "vmps_plan_workspace_bytes")
    ws = workspace if workspace is not None else _default_workspace(dev)
    buf = ws.get(int(nb.value), dev)
    mg = torch.empty((r - 1) * 4, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        rc = L.vmps_plan_from_runs(run_start.data_ptr(), r, n, mg.data_ptr(), buf.data_ptr(), buf.numel(),
                                   _stream_ptr(dev))
    _check(rc, "vmps_plan_from_runs")
    recs = mg.view(-1, 4)
    return torch.stack([recs[:, 0], recs[:, 1], recs[:, 2], recs[:, 3] & 0xFFFFFFFF], dim=1)


def sort_records(records: torch.Tensor, out: torch.Tensor | None = None, perm: bool = False,
                 workspace: Workspace | None = None):
    """vmps_sort_records: stable lexicographic sort of a (n, words) CUDA tensor
    of u32/int32 records (word 0 most significant).  Returns the sorted
    records (``out`` if given) and, with ``perm``, the permutation (uint32)."""
    if not records.is_cuda or records.dim() != 2 or not records.is_contiguous():
        raise ValueError("records must be a contiguous (n, words) CUDA tensor")
    if records.dtype not in (torch.uint32, torch.int32):
        raise ValueError("records must hold 32-bit words")
    n, words = records.shape
    dev = records.device
    res = out if out is not None else torch.empty_like(records)
    pm = torch.empty(n, dtype=torch.uint32, device=dev) if perm else None
    L = lib()
    nb = ctypes.c_size_t(0)
    _check(L.vmps_sort_records_workspace_bytes(n, words, ctypes.byref(nb)), "vmps_sort_records_workspace_bytes")
    ws = workspace if workspace is not None else _default_workspace(dev)
    buf = ws.get(int(nb.value), dev)
    with torch.cuda.device(dev):
        rc = L.vmps_sort_records(records.data_ptr(), res.data_ptr(), None if pm is None else pm.data_ptr(), n, words,
                                 buf.data_ptr(), buf.numel(), _stream_ptr(dev))
    if rc != 0:
        raise VmpsError(rc, "vmps_sort_records", L.vmps_records_last_error().decode())
    return (res, pm) if perm else res


def merge_pieces(key_ptrs: list[int], val_ptrs: list[int] | None, counts: list[int], out_keys: torch.Tensor,
                 out_values: torch.Tensor | None = None, workspace: Workspace | None = None) -> None:
    """vmps_merge_pieces: stable merge of g <= 8 sorted pieces given as device
    addresses (local tensors' data_ptr() or peer mappings from ipc_open) into
    out_keys / out_values, ties to the lower piece."""
    g = len(counts)
    kt = key_type(out_keys)
    dev = out_keys.device
    N = sum(counts)
    L = lib()
    nb = ctypes.c_size_t(0)
    _check(L.vmps_merge_pieces_workspace_bytes(N, kt, 1 if out_values is not None else 0, g, ctypes.byref(nb)),
           "vmps_merge_pieces_workspace_bytes")
    ws = workspace if workspace is not None else _default_workspace(dev)
    buf = ws.get(int(nb.value), dev)
    kp = (ctypes.c_void_p * g)(*key_ptrs)
    vpa = (ctypes.c_void_p * g)(*val_ptrs) if val_ptrs is not None else None
    cn = (ctypes.c_uint64 * g)(*counts)
    with torch.cuda.device(dev):
        rc = L.vmps_merge_pieces(kp, vpa, cn, g, out_keys.data_ptr(),
                                 None if out_values is None else out_values.data_ptr(), kt, buf.data_ptr(),
                                 buf.numel(), _stream_ptr(dev))
    _check(rc, "vmps_merge_pieces")


def ipc_handle(t: torch.Tensor) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of t's allocation, t's byte offset in it)."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_uint64(0)
    _check_comm(lib().vmps_ipc_handle(t.data_ptr(), h, ctypes.byref(off)), "vmps_ipc_handle")
    return h.raw, int(off.value)


def ipc_open(handle: bytes, offset: int) -> int:
    """Map a peer allocation (vmps_ipc_open); returns the device address."""
    p = ctypes.c_void_p()
    _check_comm(lib().vmps_ipc_open(ctypes.create_string_buffer(bytes(handle), 64), offset, ctypes.byref(p)),
                "vmps_ipc_open")
    return int(p.value)


def ipc_close(ptr: int, offset: int) -> None:
    _check_comm(lib().vmps_ipc_close(ptr, offset), "vmps_ipc_close")


# ---- native multi-GPU entry points (csrc/comm.cu) ----

def _check_comm(rc: int, where: str):
    if rc != 0:
        raise VmpsError(rc, where, lib().vmps_comm_last_error().decode())


def comm_unique_id() -> bytes:
    """vmps_comm_unique_id: 128 bytes rank 0 shares with the other ranks."""
    buf = ctypes.create_string_buffer(128)
    _check_comm(lib().vmps_comm_unique_id(buf), "vmps_comm_unique_id")
    return buf.raw


class LocalGroup:
    """A group of in-process virtual ranks (vmps_local_group_create): threads
    of this process, typically all on one GPU, that run the native protocol
    with collectives made of barriers, events and device copies."""

    def __init__(self, world: int, device: int = 0):
        self.ptr = ctypes.c_void_p()
        self.world, self.device = world, device
        _check_comm(lib().vmps_local_group_create(world, device, ctypes.byref(self.ptr)), "vmps_local_group_create")

    def destroy(self):
        if self.ptr:
            _check_comm(lib().vmps_local_group_destroy(self.ptr), "vmps_local_group_destroy")
            self.ptr = ctypes.c_void_p()


class Comm:
    """A native communicator (vmps_comm_init over NCCL, or Comm.local for a
    virtual rank of a LocalGroup); destroy() or use as a context."""

    def __init__(self, rank: int, world: int, uid: bytes | None, device: int, group: LocalGroup | None = None):
        self.ptr = ctypes.c_void_p()
        self.rank, self.world, self.device = rank, world, device
        if group is not None:
            _check_comm(lib().vmps_comm_init_local(ctypes.byref(self.ptr), rank, group.ptr, device),
                        "vmps_comm_init_local")
            return
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        _check_comm(lib().vmps_comm_init(ctypes.byref(self.ptr), rank, world, buf, device), "vmps_comm_init")

    @classmethod
    def local(cls, rank: int, group: LocalGroup) -> "Comm":
        return cls(rank, group.world, None, group.device, group)

    def destroy(self):
        if self.ptr:
            _check_comm(lib().vmps_comm_destroy(self.ptr), "vmps_comm_destroy")
            self.ptr = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.destroy()


def sort_dist_native_(comm: Comm, keys: torch.Tensor, values: torch.Tensor | None = None,
                      scratch: int | None = None, stats: bool = False, workspace: Workspace | None = None):
    """vmps_sort_*_dist: globally stable sort of the ranks' concatenated shards,
    in place (this rank keeps global output ranks [off, off + n_local))."""
    if not keys.is_cuda or not keys.is_contiguous() or keys.dim() != 1:
        raise ValueError("keys must be a contiguous 1-D CUDA tensor")
    kt = key_type(keys)
    n = keys.numel()
    sc = SCRATCH_UNBOUNDED if scratch is None else int(scratch)
    L = lib()
    nb = ctypes.c_size_t(0)
    _check(L.vmps_dist_workspace_bytes(n, kt, 1 if values is not None else 0, comm.world, sc, ctypes.byref(nb)),
           "vmps_dist_workspace_bytes")
    ws = workspace if workspace is not None else _default_workspace(keys.device)
    buf = ws.get(int(nb.value), keys.device)
    st = Stats()
    sp = ctypes.byref(st) if stats else None
    with torch.cuda.device(keys.device):
        s = _stream_ptr(keys.device)
        if values is None:
            rc = L.vmps_sort_keys_dist(comm.ptr, keys.data_ptr(), n, kt, sc, buf.data_ptr(), buf.numel(), s, sp)
        else:
            rc = L.vmps_sort_pairs_dist(comm.ptr, keys.data_ptr(), values.data_ptr(), n, kt, sc, buf.data_ptr(),
                                        buf.numel(), s, sp)
    _check_comm(rc, "vmps_sort_dist")
    return st.as_dict() if stats else None


def merge_plan_dist_native(comm: Comm, keys: torch.Tensor, n_total: int,
                           workspace: Workspace | None = None) -> Plan:
    """vmps_merge_plan_dist: this rank's runs (global positions) and the merges
    of Alg. 1's global plan whose boundary j lies in its shard."""
    kt = key_type(keys)
    n = keys.numel()
    dev = keys.device
    L = lib()
    nb = ctypes.c_size_t(0)
    _check(L.vmps_merge_plan_dist_workspace_bytes(n_total, n, kt, comm.world, ctypes.byref(nb)),
           "vmps_merge_plan_dist_workspace_bytes")
    ws = workspace if workspace is not None else _default_workspace(dev)
    buf = ws.get(int(nb.value), dev)
    c64 = ctypes.c_uint64(0)
    _check(L.vmps_merge_plan_dist_capacity(n_total, n, ctypes.byref(c64)), "vmps_merge_plan_dist_capacity")
    cap = int(c64.value)
    rs = torch.empty(cap, dtype=torch.int64, device=dev)
    rk = torch.empty(cap, dtype=torch.uint8, device=dev)
    mg = torch.empty(cap * 4, dtype=torch.int64, device=dev)
    nr, nm = ctypes.c_uint64(0), ctypes.c_uint64(0)
    with torch.cuda.device(dev):
        rc = L.vmps_merge_plan_dist(comm.ptr, keys.data_ptr(), n, kt, rs.data_ptr(), rk.data_ptr(), mg.data_ptr(),
                                    cap, ctypes.byref(nr), ctypes.byref(nm), buf.data_ptr(), buf.numel(),
                                    _stream_ptr(dev))
    _check_comm(rc, "vmps_merge_plan_dist")
    recs = mg[: 4 * int(nm.value)].view(-1, 4)
    merges = torch.stack([recs[:, 0], recs[:, 1], recs[:, 2], recs[:, 3] & 0xFFFFFFFF, recs[:, 3] >> 32], dim=1)
    return Plan(rs[: int(nr.value)], rk[: int(nr.value)], merges)


def count_rank(keys: torch.Tensor, probes: list[int]) -> tuple[torch.Tensor, torch.Tensor]:
    """vmps_count_rank: (lt, le) int64 device tensors -- the number of keys of
    the SORTED tensor whose order image is < / <= each probe image."""
    dev = keys.device
    p = torch.tensor([x - (1 << 64) if x >= (1 << 63) else x for x in probes], dtype=torch.int64, device=dev)
    lt = torch.empty(len(probes), dtype=torch.int64, device=dev)
    le = torch.empty(len(probes), dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        rc = lib().vmps_count_rank(keys.data_ptr(), keys.numel(), key_type(keys), p.data_ptr(), len(probes),
                                   lt.data_ptr(), le.data_ptr(), _stream_ptr(dev))
    _check(rc, "vmps_count_rank")
    return lt, le


def merge_runs(keys: torch.Tensor, vals: torch.Tensor | None, starts: list[int],
               workspace: Workspace | None = None) -> None:
    """vmps_merge_runs: in-place stable merge of the adjacent sorted runs that
    start at `starts` (ties to the earlier run)."""
    n = keys.numel()
    if len(starts) <= 1 or n <= 1:
        return
    kt = key_type(keys)
    L = lib()
    nb = ctypes.c_size_t(0)
    _check(L.vmps_merge_runs_workspace_bytes(n, kt, 1 if vals is not None else 0, len(starts), ctypes.byref(nb)),
           "vmps_merge_runs_workspace_bytes")
    ws = workspace if workspace is not None else _default_workspace(keys.device)
    buf = ws.get(int(nb.value), keys.device)
    hs = (ctypes.c_uint64 * len(starts))(*starts)
    with torch.cuda.device(keys.device):
        rc = L.vmps_merge_runs(keys.data_ptr(), None if vals is None else vals.data_ptr(), n, kt, hs, len(starts),
                               buf.data_ptr(), buf.numel(), _stream_ptr(keys.device))
    _check(rc, "vmps_merge_runs")


def merge_runs_bounded(keys: torch.Tensor, vals: torch.Tensor | None, starts: list[int], scratch: int,
                       workspace: Workspace | None = None) -> None:
    """vmps_merge_runs_bounded: in-place stable merge of the adjacent sorted
    runs at `starts` with the element scratch capped at `scratch`."""
    n = keys.numel()
    kt = key_type(keys)
    L = lib()
    nb = ctypes.c_size_t(0)
    _check(L.vmps_merge_runs_bounded_workspace_bytes(n, kt, 1 if vals is not None else 0, len(starts), scratch,
                                                     ctypes.byref(nb)), "vmps_merge_runs_bounded_workspace_bytes")
    ws = workspace if workspace is not None else _default_workspace(keys.device)
    buf = ws.get(int(nb.value), keys.device)
    hs = (ctypes.c_uint64 * len(starts))(*starts)
    with torch.cuda.device(keys.device):
        rc = L.vmps_merge_runs_bounded(keys.data_ptr(), None if vals is None else vals.data_ptr(), n, kt, hs,
                                       len(starts), scratch, buf.data_ptr(), buf.numel(), _stream_ptr(keys.device))
    _check(rc, "vmps_merge_runs_bounded")


def dist_cuts(comm: Comm, keys: torch.Tensor, workspace: Workspace | None = None):
    """vmps_dist_cuts on this rank's SORTED shard: (cut, sizes, rounds) with
    cut[q][t] = elements of rank q that go to ranks < t (a (g, g+1) list of
    lists) and every rank's shard size."""
    import numpy as np
    g = comm.world
    kt = key_type(keys)
    dev = keys.device
    L = lib()
    nb = ctypes.c_size_t(0)
    _check_comm(L.vmps_dist_cuts_workspace_bytes(g, ctypes.byref(nb)), "vmps_dist_cuts_workspace_bytes")
    ws = workspace if workspace is not None else _default_workspace(dev)
    buf = ws.get(int(nb.value), dev)
    cut = np.zeros(g * (g + 1), np.uint64)
    sizes = np.zeros(g, np.uint64)
    rounds = ctypes.c_uint32(0)
    with torch.cuda.device(dev):
        rc = L.vmps_dist_cuts(comm.ptr, keys.data_ptr(), keys.numel(), kt, cut.ctypes.data, sizes.ctypes.data,
                              ctypes.byref(rounds), buf.data_ptr(), buf.numel(), _stream_ptr(dev))
    _check_comm(rc, "vmps_dist_cuts")
    return cut.reshape(g, g + 1).astype(np.int64).tolist(), sizes.astype(np.int64).tolist(), int(rounds.value)


# ---- host-side protocol arithmetic of the native multi-GPU protocol (C) ----

def _u64(a):
    import numpy as np
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def splitter_probes(lo, hi):
    """vmps_splitter_probes: (probes, base) of one 16-ary search round."""
    import numpy as np
    m = len(lo)
    lo_, hi_ = _u64(lo), _u64(hi)
    pr = np.zeros(max(15 * m, 1), np.uint64)
    base = np.zeros(m + 1, np.uint32)
    nprobe = ctypes.c_uint32(0)
    _check_comm(lib().vmps_splitter_probes(m, lo_.ctypes.data, hi_.ctypes.data, pr.ctypes.data, base.ctypes.data,
                                           ctypes.byref(nprobe)), "vmps_splitter_probes")
    return [int(x) for x in pr[:nprobe.value]], [int(x) for x in base]


def splitter_update(lo, hi, R, probes, base, le_sum):
    """vmps_splitter_update: the narrowed (lo, hi) after one round."""
    import numpy as np
    m = len(lo)
    lo_, hi_ = _u64(lo), _u64(hi)
    pr, ls, r_ = _u64(probes if probes else [0]), _u64(le_sum if le_sum else [0]), _u64(R)
    b = np.ascontiguousarray(np.asarray(base, dtype=np.uint32))
    _check_comm(lib().vmps_splitter_update(m, lo_.ctypes.data, hi_.ctypes.data, r_.ctypes.data, pr.ctypes.data,
                                           b.ctypes.data, ls.ctypes.data), "vmps_splitter_update")
    return [int(x) for x in lo_], [int(x) for x in hi_]


def split_points(R: int, lt, le):
    """vmps_split_points: per-rank cut for global output rank R (ties in rank order)."""
    import numpy as np
    g = len(lt)
    out = np.zeros(g, np.uint64)
    lt_, le_ = _u64(lt), _u64(le)  # kept alive across the call
    _check_comm(lib().vmps_split_points(g, R, lt_.ctypes.data, le_.ctypes.data, out.ctypes.data),
                "vmps_split_points")
    return [int(x) for x in out]


def compose_tables(tables, sizes, ns: int):
    """vmps_compose_tables: (entry states, run counts) of consecutive shards."""
    import numpy as np
    g = len(sizes)
    t = np.zeros(g * ns, np.uint64)
    for q, tab in enumerate(tables):
        if tab is not None:
            t[q * ns:(q + 1) * ns] = np.asarray(tab, dtype=np.int64).astype(np.uint64)
    entry = np.zeros(g, np.uint32)
    count = np.zeros(g, np.uint64)
    sz_ = _u64(sizes)
    _check_comm(lib().vmps_compose_tables(g, ns, t.ctypes.data, sz_.ctypes.data, entry.ctypes.data,
                                          count.ctypes.data), "vmps_compose_tables")
    return [int(x) for x in entry], [int(x) for x in count]


def profile_enable(on: bool = True) -> None:
    """Bench hook: record CUDA events around each phase of every sort."""
    lib().vmps_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """Phase times (ms) of the last sort (its stream must be synchronised)."""
    ms = (ctypes.c_double * 5)()
    nl = (ctypes.c_uint64 * 2)()
    nb = (ctypes.c_uint64 * 3)()
    k = lib().vmps_profile_read(ms, 5, nl, nb)
    out = {"launches": int(nl[0]), "merge_launches": int(nl[1])}
    if k == 5:
        out.update(plan_ms=ms[0], leaf_ms=ms[1], partition_ms=ms[2], merge_ms=ms[3], total_ms=ms[4],
                   merge_bytes=int(nb[0]), M=int(nb[1]), fused_M=int(nb[2]))
    return out


def test_set_minrun(m: int) -> None:
    """Test hook: force minrun (0 = the paper's rule)."""
    lib().vmps_test_set_minrun(m)


def test_set_mode(levels_per_pass: int = 2) -> None:
    """Test hook: tree levels merged per HBM pass, 2 (default, 4-way merges) or 1."""
    lib().vmps_test_set_mode(int(levels_per_pass))


def test_set_leaf(radix: bool = False) -> None:
    """Test hook: leaf engine = LSD radix sort (True) or block merge sort (default)."""
    lib().vmps_test_set_leaf(1 if radix else 0)


def test_set_tiles(fuse_z: int = 0, merge_tile: int = 0, block_elems: int = 0) -> None:
    """Test hook: shrink fused-subtree / merge-tile / bounded-block sizes (0 = default)."""
    lib().vmps_test_set_tiles(fuse_z, merge_tile, block_elems)


def test_set_bd_chunk(chunk: int = 0) -> None:
    """Test hook: chunk of the chunked scratch-bounded mode (0 = 2^24)."""
    lib().vmps_test_set_bd_chunk(chunk)
