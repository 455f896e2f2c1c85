"""GPU parity of the distributed merge plan: the plan of
the concatenation of g shards, each shard processed on its own by the real
kernels (vmps_shard_chain / vmps_shard_runs, host composition of the transfer
tables, vmps_plan_from_runs), vs the oracle's plan-only pass over the whole
array -- run starts, kinds and the merge records, exact.  g virtual ranks on
one GPU run the library's own protocol (vmps_merge_plan_dist over a
vmps_local_group, tests/vranks.py): each rank's runs and merges are its part
of the whole plan.

Cuts are placed where the chain is hardest: inside long ascending and
strictly descending runs, inside a minrun-forced extension, on run-detection
tile boundaries (multiples of 4096), and shards shorter than the halo."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vm():
    import paper_2605_27147_b200 as vm
    assert torch.cuda.is_available()
    vm.lib()
    vm.test_set_minrun(0)
    return vm


def _runs_array(rng, n, dtype, desc_p=0.4, nseg=None):
    x = rng.integers(0, 1 << 20, n)
    nseg = nseg if nseg is not None else max(2, n // 300)
    cuts = np.sort(rng.integers(0, n + 1, nseg))
    for a, b in zip(cuts[:-1], cuts[1:]):
        if rng.random() < desc_p:
            x[a:b] = np.sort(x[a:b])[::-1]
        elif rng.random() < 0.7:
            x[a:b] = np.sort(x[a:b])
    if dtype == np.float32:
        return (x.astype(np.float64) / 7.0 - 5000.0).astype(np.float32)
    if dtype == np.uint64:
        return (x.astype(np.uint64) << np.uint64(31)) | np.uint64(5)
    return x.astype(np.uint32)


class _Res:
    pass


def _check(vm, glob, cuts):
    from tests import vranks
    edges = [0] + sorted(cuts) + [len(glob)]
    shards = [glob[a:b].copy() for a, b in zip(edges[:-1], edges[1:])]
    n = len(glob)

    def fn(rank, comm):
        p = vm.merge_plan_dist_native(comm, W.from_numpy(shards[rank], "cuda"), n)
        return p.run_start.cpu().numpy(), p.run_kind.cpu().numpy(), p.merges.cpu().numpy()

    outs = vranks.run(len(shards), fn)
    oplan, _ = oracle.plan(glob)
    ors = oplan.run_start.astype(np.int64)
    got = np.concatenate([o[0] for o in outs])
    assert len(got) == len(ors), f"run count {len(got)} vs {len(ors)}"
    assert (got == ors).all(), "run starts differ"
    assert (np.concatenate([o[1] for o in outs]) == oplan.run_kind).all(), "run kinds differ"
    om = np.stack([oplan.merges["i"], oplan.merges["j"], oplan.merges["k"], oplan.merges["power"]],
                  axis=1).astype(np.int64)
    ms = [o[2] for o in outs if len(o[2])]
    mg = np.concatenate(ms) if ms else np.zeros((0, 5), np.int64)
    mg = mg[np.argsort(mg[:, 4], kind="stable")]
    assert (mg[:, 4] == np.arange(len(om))).all(), "execution ranks differ"
    assert (mg[:, :4] == om).all(), "merge plan differs"
    res = _Res()
    res.counts = [len(o[0]) for o in outs]
    for q, (a, b) in enumerate(zip(edges[:-1], edges[1:])):
        assert res.counts[q] == int(((ors >= a) & (ors < b)).sum())
    res.run_start = torch.from_numpy(got)
    res.merges = torch.from_numpy(mg[:, :4].copy())
    return res


@pytest.mark.parametrize("dtype", [np.uint32, np.uint64, np.float32])
@pytest.mark.parametrize("n,g,seed", [(5000, 2, 1), (200_000, 5, 2), (3_000_003, 8, 3)])
def test_random_cuts(vm, dtype, n, g, seed):
    rng = np.random.default_rng(seed)
    glob = _runs_array(rng, n, dtype)
    cuts = sorted(set(int(c) for c in rng.integers(1, n, g - 1)))
    _check(vm, glob, cuts)


def test_single_shard_matches_merge_plan(vm):
    rng = np.random.default_rng(4)
    glob = _runs_array(rng, 100_000, np.uint32)
    res = _check(vm, glob, [])
    p = vm.merge_plan(W.from_numpy(glob, "cuda"))
    assert (p.merges.cpu() == res.merges.cpu()).all()


@pytest.mark.parametrize("dtype", [np.uint32, np.uint64])
def test_cuts_inside_runs(vm, dtype):
    """Cuts one key into, in the middle of and one key before the end of long
    ascending / strictly descending runs and of minrun-forced extensions."""
    rng = np.random.default_rng(5)
    n = 60_000
    x = rng.integers(0, 1 << 20, n)
    x[1000:9000] = np.sort(x[1000:9000])            # long ascending
    x[9000:20000] = np.sort(x[9000:20000])[::-1]    # long descending (ties possible: split)
    x[20000:20010] = np.arange(20010, 20000, -1)    # short strictly descending (extended)
    x[30000:50000] = np.arange(50000, 30000, -1)    # long strictly descending
    glob = x.astype(np.uint64) << np.uint64(20) if dtype == np.uint64 else x.astype(np.uint32)
    for cuts in ([1001], [5000], [8999], [9001], [15000], [19999], [20001], [20005],
                 [30001, 40000, 49999], [4096, 8192, 3 * 4096, 10 * 4096]):
        _check(vm, glob, cuts)


def test_tiny_shards_and_edges(vm):
    """Shards of 1..3 keys (shorter than the halo: the halo spans several
    shards), first / last shard of one key, cuts on tile boundaries."""
    rng = np.random.default_rng(6)
    n = 50_000
    glob = _runs_array(rng, n, np.uint32, nseg=100)
    _check(vm, glob, [1, 2, 3, 5, 8, 13, 4096, 4097, 8192, n - 3, n - 2, n - 1])
    _check(vm, glob, [k * 4096 for k in range(1, 12)])
    _check(vm, glob, list(range(100, 400, 3)))  # 100 shards of 3 keys in a row


@pytest.mark.parametrize("kind", ["sorted", "reversed", "equal", "sawtooth"])
def test_degenerate_arrays(vm, kind):
    n = 100_000
    if kind == "sorted":
        glob = np.arange(n, dtype=np.uint32)
    elif kind == "reversed":
        glob = np.arange(n, 0, -1).astype(np.uint32)
    elif kind == "equal":
        glob = np.full(n, 7, np.uint32)
    else:
        glob = (np.arange(n) % 37).astype(np.uint32)
    _check(vm, glob, [7, 4096, 33333, 33334, 99_999])


def test_large_sharded(vm):
    """2^24 keys (cfg2's size) in 8 shards of unequal size."""
    glob = W.to_numpy(W.make(2, n=1 << 24)[0])
    rng = np.random.default_rng(7)
    cuts = sorted(set(int(c) for c in rng.integers(1, len(glob), 7)))
    _check(vm, glob, cuts)


@pytest.mark.parametrize("N,r", [((1 << 33) + 12345, 200_003), ((1 << 36) - 7, 50_000), (10 ** 9 + 7, 1)])
def test_plan_from_runs_global_n(vm, N, r):
    """vmps_plan_from_runs on 64-bit global positions (the concatenation of
    shards can exceed 2^32 elements) vs the oracle's Alg. 1 policy on the
    same run starts (powers P:445-446 with the global n)."""
    rng = np.random.default_rng(r)
    if r == 1:
        starts = np.array([0], np.uint64)
    else:
        cuts = np.unique(rng.integers(1, N, r - 1, dtype=np.uint64))
        starts = np.concatenate([[0], cuts]).astype(np.uint64)
    d = torch.from_numpy(np.concatenate([starts, [N]]).astype(np.int64)).cuda()
    got = vm.plan_from_runs(d, N).cpu().numpy()
    mg, _ = oracle.policy(N, starts)
    want = np.stack([mg["i"], mg["j"], mg["k"], mg["power"]], axis=1).astype(np.int64) if len(mg) else \
        np.zeros((0, 4), np.int64)
    assert got.shape == want.shape and (got == want).all()
