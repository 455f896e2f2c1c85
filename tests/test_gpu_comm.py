"""GPU tests of the native multi-GPU entry points (csrc/comm.cu) through the
C ABI, at world size 1 (one GPU per process; NCCL refuses two ranks on one
device): vmps_sort_*_dist equals the oracle's stable sort, vmps_merge_plan_dist
equals the oracle's plan (every run and merge belongs to the single shard,
`order` = execution rank), and the workspace / argument errors.  The
multi-rank protocol logic is exercised with gloo in tests/test_dist.py."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    import paper_2605_27147_b200 as vm
    assert torch.cuda.is_available()
    vm.test_set_minrun(0)
    c = vm.Comm(0, 1, vm.comm_unique_id(), 0)
    yield c
    c.destroy()


@pytest.mark.parametrize("dtype,payload", [(np.uint32, True), (np.uint64, True), (np.float32, False)])
def test_sort_dist_world1(comm, dtype, payload):
    import paper_2605_27147_b200 as vm
    rng = np.random.default_rng(11)
    n = 300_001
    if dtype == np.float32:
        k = rng.standard_normal(n).astype(np.float32)
        k[rng.random(n) < 0.01] = -0.0
        k[rng.random(n) < 0.01] = np.nan
    elif dtype == np.uint64:
        k = (rng.integers(0, 16, n).astype(np.uint64) << np.uint64(33))
    else:
        k = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        k[1000:50000] = np.sort(k[1000:50000])
    v = np.arange(n, dtype=np.uint32) if payload else None
    ko, vo, _, _ = oracle.sort(k, v)
    kd = W.from_numpy(k, "cuda")
    vd = W.from_numpy(v, "cuda") if payload else None
    vm.sort_dist_native_(comm, kd, vd)
    torch.cuda.synchronize()
    assert W.to_numpy(kd).view(np.uint8).tobytes() == ko.view(np.uint8).tobytes()
    if payload:
        assert (W.to_numpy(vd) == vo).all()


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_merge_plan_dist_world1(comm, cfg):
    import paper_2605_27147_b200 as vm
    n = {1: 1 << 18, 2: 1 << 20, 3: 1 << 19}[cfg]
    keys = W.make(cfg, n=n)[0]
    kn = W.to_numpy(keys)
    oplan, _ = oracle.plan(kn)
    p = vm.merge_plan_dist_native(comm, W.from_numpy(kn, "cuda"), n)
    torch.cuda.synchronize()
    assert (p.run_start.cpu().numpy() == oplan.run_start.astype(np.int64)).all()
    assert (p.run_kind.cpu().numpy() == oplan.run_kind).all()
    om = np.stack([oplan.merges["i"], oplan.merges["j"], oplan.merges["k"], oplan.merges["power"],
                   np.arange(len(oplan.merges))], axis=1).astype(np.int64)
    assert (p.merges.cpu().numpy() == om).all()


def test_dist_errors(comm):
    import ctypes
    import paper_2605_27147_b200 as vm
    L = vm.lib()
    k = torch.zeros(1024, dtype=torch.uint32, device="cuda")
    small = torch.empty(256, dtype=torch.uint8, device="cuda")
    rc = L.vmps_sort_keys_dist(comm.ptr, k.data_ptr(), 1024, vm.KEY_U32, -1, small.data_ptr(), 256, None, None)
    assert rc == vm.ERR_BUDGET
    rc = L.vmps_sort_keys_dist(None, k.data_ptr(), 1024, vm.KEY_U32, -1, small.data_ptr(), 256, None, None)
    assert rc == vm.ERR_INVALID_ARG
    nb = ctypes.c_size_t(0)
    assert L.vmps_dist_workspace_bytes(1024, vm.KEY_U32, 0, 0, -1, ctypes.byref(nb)) == vm.ERR_INVALID_ARG
