"""GPU tests of the multi-GPU building blocks through the C ABI:
vmps_count_rank vs NumPy searchsorted on the order image, vmps_merge_runs vs
the oracle, and the whole sharded protocol with g virtual ranks on one GPU
(collectives replaced by in-process concatenation; device ops are the real
kernels)."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
from tests import refcheck as R
from tests.test_dist import image_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vm():
    import paper_2605_27147_b200 as vm
    assert torch.cuda.is_available()
    vm.lib()
    return vm


@pytest.mark.parametrize("dtype", [np.uint32, np.uint64, np.float32])
def test_count_rank(vm, dtype):
    from paper_2605_27147_b200.dist import VmpsOps
    rng = np.random.default_rng(1)
    n = 100003
    if dtype == np.float32:
        a = rng.choice(np.array([0.0, -0.0, 1.0, -3.0, np.nan, np.inf], np.float32), n)
    else:
        a = rng.integers(0, 50, n).astype(dtype)
    img = image_np(a)
    idx = np.argsort(img, kind="stable")
    a = a[idx]
    img = img[idx]
    probes = sorted(set(int(x) for x in img[rng.integers(0, n, 50)])) + [0, int(img.max()) + 1]
    lt, le = VmpsOps().count(W.from_numpy(a, "cuda"), probes)
    p = np.array(probes, dtype=np.uint64)
    assert (lt.cpu().numpy() == np.searchsorted(img, p, "left")).all()
    assert (le.cpu().numpy() == np.searchsorted(img, p, "right")).all()


@pytest.mark.parametrize("dtype", [np.uint32, np.uint64, np.float32])
@pytest.mark.parametrize("pieces", [2, 3, 5, 8])
def test_merge_runs(vm, dtype, pieces):
    from paper_2605_27147_b200.dist import VmpsOps
    rng = np.random.default_rng(pieces)
    sizes = rng.integers(1, 40000, pieces)
    ks, starts, acc = [], [], 0
    for s in sizes:
        if dtype == np.float32:
            k = rng.choice(np.array([0.0, -0.0, 1.0, -3.0, np.nan], np.float32), s)
        else:
            k = rng.integers(0, 9, s).astype(dtype)
        ks.append(k[np.argsort(image_np(k), kind="stable")])
        starts.append(acc)
        acc += s
    keys = np.concatenate(ks)
    vals = np.arange(acc, dtype=np.uint32)
    gk, gv = W.from_numpy(keys, "cuda"), W.from_numpy(vals, "cuda")
    VmpsOps().merge_runs(gk, gv, starts)
    torch.cuda.synchronize()
    ek, ev = R.stable_sorted(keys)
    assert W.to_numpy(gk).view(np.uint8).tobytes() == ek.view(np.uint8).tobytes()
    assert (W.to_numpy(gv) == ev).all()


def test_sharded_protocol_virtual_ranks(vm):
    """sort_dist's steps with 4 virtual ranks on one GPU: real kernels for the
    local sorts, counts and final merges; the collectives are in-process."""
    from paper_2605_27147_b200.dist import VmpsOps, split_points
    ops = VmpsOps()
    g, n = 4, 1 << 18
    shards = [W.cfg5(n=n, device="cuda", rank=q) for q in range(g)]
    allk = np.concatenate([W.to_numpy(k) for k, _ in shards])
    allv = np.concatenate([W.to_numpy(v) for _, v in shards])
    for k, v in shards:
        ops.local_sort(k, v)
    N = g * n
    Rt = [t * N // g for t in range(1, g)]
    lo, hi = [0] * (g - 1), [(1 << 32) - 1] * (g - 1)
    while any(a < b for a, b in zip(lo, hi)):
        mid = [(a + b) // 2 for a, b in zip(lo, hi)]
        le = sum(ops.count(k, mid)[1].cpu() for k, _ in shards).tolist()
        for t in range(g - 1):
            if lo[t] < hi[t]:
                if le[t] >= Rt[t]:
                    hi[t] = mid[t]
                else:
                    lo[t] = mid[t] + 1
    cnt = [ops.count(k, lo) for k, _ in shards]
    cut = [[0] + [0] * (g - 1) + [n] for _ in range(g)]
    for t in range(g - 1):
        pts = split_points(Rt[t], [int(c[0][t]) for c in cnt], [int(c[1][t]) for c in cnt])
        for q in range(g):
            cut[q][t + 1] = pts[q]
    outk, outv = [], []
    for p in range(g):
        pk = torch.cat([shards[q][0][cut[q][p]:cut[q][p + 1]] for q in range(g)])
        pv = torch.cat([shards[q][1][cut[q][p]:cut[q][p + 1]] for q in range(g)])
        sizes = [cut[q][p + 1] - cut[q][p] for q in range(g)]
        starts, acc = [], 0
        for c in sizes:
            if c:
                starts.append(acc)
            acc += c
        ops.merge_runs(pk, pv, starts)
        outk.append(W.to_numpy(pk))
        outv.append(W.to_numpy(pv))
    ko, vo, _, _ = oracle.sort(allk, allv)
    assert (np.concatenate(outk) == ko).all()
    assert (np.concatenate(outv) == vo).all()
