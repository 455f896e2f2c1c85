"""GPU tests of the multi-GPU building blocks through the C ABI:
vmps_count_rank vs NumPy searchsorted on the order image, vmps_merge_runs vs
the oracle.  The whole sharded protocol with g virtual ranks on one GPU runs
in tests/test_gpu_comm.py."""
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
    lt, le = vm.count_rank(W.from_numpy(a, "cuda"), probes)
    p = np.array(probes, dtype=np.uint64)
    assert (lt.cpu().numpy() == np.searchsorted(img, p, "left")).all()
    assert (le.cpu().numpy() == np.searchsorted(img, p, "right")).all()


@pytest.mark.parametrize("dtype", [np.uint32, np.uint64, np.float32])
@pytest.mark.parametrize("pieces", [2, 3, 5, 8])
def test_merge_runs(vm, dtype, pieces):
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
    vm.merge_runs(gk, gv, starts)
    torch.cuda.synchronize()
    ek, ev = R.stable_sorted(keys)
    assert W.to_numpy(gk).view(np.uint8).tobytes() == ek.view(np.uint8).tobytes()
    assert (W.to_numpy(gv) == ev).all()
