"""GPU tests of the native multi-GPU entry points (csrc/comm.cu) through the
C ABI: at world size 1 over NCCL (one GPU per process; NCCL refuses two ranks
on one device), and with g = 2..8 virtual ranks on one GPU (threads of this
process, vmps_local_group: the same protocol, collectives over barriers,
events and device copies).  vmps_sort_*_dist equals the oracle's stable sort
of the concatenated shards (rank p keeps global output ranks [off_p, off_p +
n_p)), vmps_merge_plan_dist's per-rank pieces are the oracle's plan of the
whole array, vmps_dist_cuts' table matches its definition; a rank that never
joins makes the others fail with VMPS_ERR_NCCL after the timeout."""
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


# ---- virtual ranks: the native protocol with g ranks on one GPU ----

def _shards(rng, sizes, dtype):
    out = []
    for n in sizes:
        if dtype == np.float32:
            k = rng.standard_normal(n).astype(np.float32)
            m = rng.random(n) < 0.3  # ties, signed zeros and NaNs across shards
            k[m] = rng.choice(np.array([0.0, -0.0, 1.5, -2.0, np.nan, 3.0], np.float32), int(m.sum()))
        elif dtype == np.uint64:
            k = (rng.integers(0, 9, n).astype(np.uint64) << np.uint64(40)) | rng.integers(0, 3, n).astype(np.uint64)
        else:
            k = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
            k[: n // 3] = rng.integers(0, 7, n // 3)  # ties across shards
            k[n // 3: n // 2] = np.sort(k[n // 3: n // 2])
        out.append(k)
    return out


@pytest.mark.parametrize("g,dtype,sizes", [
    (2, np.uint32, [200_000, 150_001]),
    (3, np.uint64, [70_000, 0, 123_457]),          # an empty shard
    (4, np.float32, [50_000, 50_000, 3, 90_000]),  # a tiny shard
    (8, np.uint32, [40_000 + 1000 * q for q in range(8)]),
])
def test_sort_dist_virtual_ranks(g, dtype, sizes):
    import paper_2605_27147_b200 as vm
    from tests import vranks
    rng = np.random.default_rng(g * 7 + len(sizes))
    ks = _shards(rng, sizes, dtype)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    vs = [np.arange(offs[q], offs[q + 1], dtype=np.uint32) for q in range(g)]

    def fn(rank, comm):
        kd = W.from_numpy(ks[rank], "cuda")
        vd = W.from_numpy(vs[rank], "cuda")
        vm.sort_dist_native_(comm, kd, vd)
        return W.to_numpy(kd), W.to_numpy(vd)

    outs = vranks.run(g, fn)
    ko, vo, _, _ = oracle.sort(np.concatenate(ks), np.concatenate(vs))
    for q in range(g):
        assert len(outs[q][0]) == sizes[q]
    assert np.concatenate([o[0] for o in outs]).view(np.uint8).tobytes() == ko.view(np.uint8).tobytes()
    assert (np.concatenate([o[1] for o in outs]) == vo).all()


def test_sort_dist_virtual_ranks_cfg5():
    """cfg5-shaped shards (2^20 per rank, 4 ranks, payload = global index), keys only and pairs."""
    import paper_2605_27147_b200 as vm
    from tests import vranks
    g, n = 4, 1 << 20
    sh = [W.cfg5(n=n, device="cpu", rank=q) for q in range(g)]
    ks = [W.to_numpy(k) for k, _ in sh]
    vs = [W.to_numpy(v) for _, v in sh]

    def fn(rank, comm):
        kd = W.from_numpy(ks[rank], "cuda")
        vd = W.from_numpy(vs[rank], "cuda")
        vm.sort_dist_native_(comm, kd, vd)
        k2 = W.from_numpy(ks[rank], "cuda")
        vm.sort_dist_native_(comm, k2)
        return W.to_numpy(kd), W.to_numpy(vd), W.to_numpy(k2)

    outs = vranks.run(g, fn)
    ko, vo, _, _ = oracle.sort(np.concatenate(ks), np.concatenate(vs))
    assert (np.concatenate([o[0] for o in outs]) == ko).all()
    assert (np.concatenate([o[1] for o in outs]) == vo).all()
    assert (np.concatenate([o[2] for o in outs]) == ko).all()


@pytest.mark.parametrize("g,n,seed", [(2, 300_000, 1), (5, 1_000_003, 2), (8, 2_000_000, 3)])
def test_merge_plan_dist_virtual_ranks(g, n, seed):
    """Each rank's runs and merges (j in its shard) are exactly its part of the
    oracle's plan of the whole array, with the global execution rank."""
    import paper_2605_27147_b200 as vm
    from tests import vranks
    rng = np.random.default_rng(seed)
    x = rng.integers(0, 1 << 20, n)
    cuts = np.sort(rng.integers(0, n, max(2, n // 500)))
    for a, b in zip(cuts[:-1], cuts[1:]):
        x[a:b] = np.sort(x[a:b])[::-1] if rng.random() < 0.3 else np.sort(x[a:b])
    glob = x.astype(np.uint32)
    edges = [0] + sorted(set(int(c) for c in rng.integers(1, n, g - 1))) + [n]
    while len(edges) < g + 1:
        edges.insert(1, edges[1])  # repeated cut: an empty shard
    shards = [glob[a:b].copy() for a, b in zip(edges[:-1], edges[1:])]

    def fn(rank, comm):
        p = vm.merge_plan_dist_native(comm, W.from_numpy(shards[rank], "cuda"), n)
        return p.run_start.cpu().numpy(), p.run_kind.cpu().numpy(), p.merges.cpu().numpy()

    outs = vranks.run(g, fn)
    oplan, _ = oracle.plan(glob)
    rs = np.concatenate([o[0] for o in outs])
    rk = np.concatenate([o[1] for o in outs])
    assert (rs == oplan.run_start.astype(np.int64)).all()
    assert (rk == oplan.run_kind).all()
    mg = np.concatenate([o[2] for o in outs if len(o[2])])
    mg = mg[np.argsort(mg[:, 4])]
    om = np.stack([oplan.merges["i"], oplan.merges["j"], oplan.merges["k"], oplan.merges["power"]], axis=1)
    assert (mg[:, 4] == np.arange(len(om))).all()
    assert (mg[:, :4] == om.astype(np.int64)).all()


def test_dist_cuts_virtual_ranks():
    """vmps_dist_cuts on sorted shards: every rank gets the same table, whose
    column t sums to off_t and whose pieces are exactly the global ranks."""
    import paper_2605_27147_b200 as vm
    from tests import vranks
    g = 3
    rng = np.random.default_rng(5)
    sizes = [5000, 7000, 4000]
    ks = [np.sort(rng.integers(0, 50, s).astype(np.uint32)) for s in sizes]

    def fn(rank, comm):
        return vm.dist_cuts(comm, W.from_numpy(ks[rank], "cuda"))

    outs = vranks.run(g, fn)
    cut, szs, rounds = outs[0]
    assert all(o[0] == cut and o[1] == sizes for o in outs)
    off = np.concatenate([[0], np.cumsum(sizes)])
    allk = np.concatenate(ks)
    order = np.argsort(allk, kind="stable")
    owner = np.concatenate([np.full(s, q) for q, s in enumerate(sizes)])
    local = np.concatenate([np.arange(s) for s in sizes])
    for t in range(g + 1):
        assert sum(cut[q][t] for q in range(g)) == off[t]
    for p in range(g):  # rank p's output = its pieces, in global stable order
        got = sorted((q, i) for q in range(g) for i in range(cut[q][p], cut[q][p + 1]))
        want = sorted(zip(owner[order[off[p]:off[p + 1]]], local[order[off[p]:off[p + 1]]]))
        assert got == want


def test_virtual_rank_timeout(monkeypatch):
    """A rank that never joins the collective: the others return
    VMPS_ERR_NCCL (5) after VMPS_COMM_TIMEOUT_S instead of hanging."""
    import threading

    import paper_2605_27147_b200 as vm
    monkeypatch.setenv("VMPS_COMM_TIMEOUT_S", "2")
    group = vm.LocalGroup(2, 0)
    c0 = vm.Comm.local(0, group)
    res = {}

    def body():
        try:
            kd = torch.arange(10000, 0, -1, dtype=torch.int32, device="cuda").view(torch.uint32)
            vm.sort_dist_native_(c0, kd)
        except vm.VmpsError as e:
            res["status"] = e.status
            res["msg"] = str(e)

    t = threading.Thread(target=body)
    t.start()
    t.join(60)
    assert not t.is_alive()
    assert res.get("status") == 5, res
    c0.destroy()
    group.destroy()


# ---- scratch-bounded multi-GPU sort: cap per rank, exchange staging included ----

@pytest.mark.parametrize("g,dtype,sizes,minrun", [
    (2, np.uint32, [150_000, 120_001], 0),
    (3, np.uint64, [40_000, 0, 70_003], 0),          # an empty shard
    (4, np.float32, [30_000, 12_000, 45_000, 20_000], 0),  # unequal shards
    (4, np.uint32, [60_000] * 4, 4),                  # many runs (minrun 4)
])
def test_sort_dist_bounded_virtual_ranks(g, dtype, sizes, minrun):
    """vmps_sort_pairs_dist with scratch_elems = 4 sqrt(n log2 n) per rank:
    identical to the oracle's stable sort of the concatenation; the element
    scratch (the local sorts' blocks and the swap staging) stays within the cap."""
    import math

    import paper_2605_27147_b200 as vm
    from tests import vranks
    rng = np.random.default_rng(31 * g + len(sizes))
    ks = _shards(rng, sizes, dtype)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    vs = [np.arange(offs[q], offs[q + 1], dtype=np.uint32) for q in range(g)]
    caps = [int(4 * math.sqrt(max(s, 2) * math.log2(max(s, 2)))) for s in sizes]
    caps = [max(c, 6 * 64) for c in caps]
    vm.test_set_minrun(minrun)
    try:
        def fn(rank, comm):
            kd = W.from_numpy(ks[rank], "cuda")
            vd = W.from_numpy(vs[rank], "cuda")
            st = vm.sort_dist_native_(comm, kd, vd, scratch=caps[rank], stats=True)
            return W.to_numpy(kd), W.to_numpy(vd), st

        outs = vranks.run(g, fn)
    finally:
        vm.test_set_minrun(0)
    ko, vo, _, _ = oracle.sort(np.concatenate(ks), np.concatenate(vs))
    for q in range(g):
        assert len(outs[q][0]) == sizes[q]
    assert np.concatenate([o[0] for o in outs]).view(np.uint8).tobytes() == ko.view(np.uint8).tobytes()
    assert (np.concatenate([o[1] for o in outs]) == vo).all()
    w = np.dtype(dtype).itemsize + 4
    for q in range(g):
        st = outs[q][2]
        if sizes[q] > 1:
            assert st["scratch_bytes"] <= caps[q] * w, (q, st["scratch_bytes"], caps[q] * w)


def test_sort_dist_bounded_cfg5_virtual_ranks():
    """cfg5-shaped shards, 2^20 per rank, 2 ranks, the cap 4 sqrt(n log2 n)."""
    import math

    import paper_2605_27147_b200 as vm
    from tests import vranks
    g, n = 2, 1 << 20
    sh = [W.cfg5(n=n, device="cpu", rank=q) for q in range(g)]
    ks = [W.to_numpy(k) for k, _ in sh]
    vs = [W.to_numpy(v) for _, v in sh]
    S = int(4 * math.sqrt(n * math.log2(n)))

    def fn(rank, comm):
        kd = W.from_numpy(ks[rank], "cuda")
        vd = W.from_numpy(vs[rank], "cuda")
        st = vm.sort_dist_native_(comm, kd, vd, scratch=S, stats=True)
        return W.to_numpy(kd), W.to_numpy(vd), st

    outs = vranks.run(g, fn)
    ko, vo, _, _ = oracle.sort(np.concatenate(ks), np.concatenate(vs))
    assert (np.concatenate([o[0] for o in outs]) == ko).all()
    assert (np.concatenate([o[1] for o in outs]) == vo).all()
    assert all(o[2]["scratch_bytes"] <= S * 8 for o in outs)
