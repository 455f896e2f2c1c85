"""GPU parity of the pull-merge: vmps_merge_pieces merges g
sorted pieces that live at arbitrary device addresses (separate allocations,
and misaligned sub-ranges of one allocation -- the TMA windows are aligned
down / up inside them) into one output, ties to the lower piece; compared
with the oracle's stable sort of the concatenated pieces (exact: a stable
sort of sorted pieces is their stable merge in piece order).  Also the
protocol dist.sort_dist_pull at world size 1 over NCCL (multi-rank peer
mappings need one GPU per rank)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


def _pieces(rng, g, dtype, n_max):
    ps = []
    for q in range(g):
        n = int(rng.integers(0, n_max)) if rng.random() < 0.85 else 0
        if dtype == np.float32:
            pool = np.array([0.0, -0.0, 1.0, -1.0, np.nan, np.inf, -np.inf, 2.5], np.float32)
            x = pool[rng.integers(0, len(pool), n)] if rng.random() < 0.5 else rng.standard_normal(n).astype(np.float32)
            img = x.view(np.uint32).astype(np.int64)
            nan = (img & 0x7FFFFFFF) > 0x7F800000
            key = np.where(nan, 0xFFFFFFFF, np.where(img >> 31, img ^ 0xFFFFFFFF, img | 0x80000000))
            x = x[np.argsort(key, kind="stable")]
        elif dtype == np.uint64:
            x = np.sort(rng.integers(0, 6, n).astype(np.uint64) << np.uint64(40))
        else:
            x = np.sort(rng.integers(0, 1000, n).astype(np.uint32))
        ps.append(x)
    return ps


@pytest.mark.parametrize("dtype", [np.uint32, np.uint64, np.float32])
@pytest.mark.parametrize("g", [1, 2, 3, 4, 5, 8])
def test_merge_pieces(dtype, g):
    import paper_2605_27147_b200 as vm
    rng = np.random.default_rng(g * 10 + (dtype == np.uint64) + 2 * (dtype == np.float32))
    for trial in range(4):
        ps = _pieces(rng, g, dtype, 30000 if trial < 3 else 300)
        counts = [len(p) for p in ps]
        N = sum(counts)
        if N == 0:
            continue
        allk = np.concatenate(ps)
        allv = np.arange(N, dtype=np.uint32)
        # trial 0: separate allocations; otherwise sub-ranges of one buffer at odd offsets
        if trial == 0:
            tk = [W.from_numpy(p, "cuda") if len(p) else torch.empty(0, device="cuda") for p in ps]
            kptr = [t.data_ptr() if t.numel() else 0 for t in tk]
            offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
            tv = [torch.from_numpy(allv[offs[q]:offs[q + 1]].view(np.int32).copy()).cuda() for q in range(g)]
            vptr = [t.data_ptr() if t.numel() else 0 for t in tv]
        else:
            pad = 3
            big = np.zeros(N + pad * g + 8, dtype=allk.dtype)
            bigv = np.zeros(N + pad * g + 8, dtype=np.uint32)
            starts, pos = [], 1
            for q, p in enumerate(ps):
                starts.append(pos)
                big[pos:pos + len(p)] = p
                o = sum(counts[:q])
                bigv[pos:pos + len(p)] = allv[o:o + len(p)]
                pos += len(p) + pad
            tkb = W.from_numpy(big, "cuda")
            tvb = torch.from_numpy(bigv.view(np.int32)).cuda()
            kptr = [tkb.data_ptr() + s * big.itemsize for s in starts]
            vptr = [tvb.data_ptr() + s * 4 for s in starts]
        ok = torch.empty(N, dtype=W.from_numpy(allk[:1]).dtype, device="cuda")
        ov = torch.empty(N, dtype=torch.uint32, device="cuda")
        vm.merge_pieces(kptr, vptr, counts, ok, ov)
        torch.cuda.synchronize()
        ko, vo, _, _ = oracle.sort(allk, allv)
        assert W.to_numpy(ok).view(np.uint8).tobytes() == ko.view(np.uint8).tobytes(), (g, trial)
        assert (ov.cpu().view(torch.int32).numpy().view(np.uint32) == vo).all(), (g, trial)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sort_dist_pull_world1():
    import torch.distributed as dist
    from paper_2605_27147_b200.dist import sort_dist_pull
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        k, v = W.cfg5(n=1 << 20, device="cuda")
        k0, v0 = W.to_numpy(k), W.to_numpy(v)
        res = sort_dist_pull(k, v)
        torch.cuda.synchronize()
        ko, vo, _, _ = oracle.sort(k0, v0)
        assert (W.to_numpy(res.keys) == ko).all() and (W.to_numpy(res.vals) == vo).all()
    finally:
        dist.destroy_process_group()
