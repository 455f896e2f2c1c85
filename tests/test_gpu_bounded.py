"""Scratch-bounded mode: same output as the unbounded mode and
the oracle, element scratch within the cap c*sqrt(n log2 n) (reading R7),
peak bytes reported; small blocks and tiny caps force many rounds, block
evictions and a long final Copy."""
import math

import numpy as np
import pytest
import torch

import oracle
import workloads as W
from tests.test_gpu_parity import _structured, check_case  # noqa: F401  (fixtures reuse)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vm():
    import paper_2605_27147_b200 as vm
    assert torch.cuda.is_available()
    vm.lib()
    yield vm
    vm.test_set_minrun(0)
    vm.test_set_tiles(0, 0, 0)


def cap(n, c=4):
    return int(c * math.sqrt(n * math.log2(n)))


def bounded_vs_oracle(vm, keys, vals, scratch, minrun=0):
    vm.test_set_minrun(minrun)
    ko, vo, _, ost = oracle.sort(keys, vals, minrun_override=minrun)
    k = W.from_numpy(keys, "cuda")
    v = None if vals is None else W.from_numpy(vals, "cuda")
    st = vm.sort_(k, v, scratch=scratch, stats=True)
    torch.cuda.synchronize()
    assert W.to_numpy(k).view(np.uint8).tobytes() == ko.view(np.uint8).tobytes(), "keys differ"
    if vals is not None:
        assert (W.to_numpy(v) == vo).all(), "payload differs"
    assert st["merge_cost_M"] == ost["merge_cost_M"]
    w = keys.dtype.itemsize + (4 if vals is not None else 0)
    assert st["scratch_bytes"] <= scratch * w, (st["scratch_bytes"], scratch * w)
    assert st["block_elems"] > 0
    return st


@pytest.mark.parametrize("dtype", [np.uint32, np.uint64, np.float32])
def test_bounded_tiny_blocks(vm, dtype):
    rng = np.random.default_rng(300 + (dtype == np.uint64) + 2 * (dtype == np.float32))
    try:
        for trial in range(30):
            blk = int(rng.choice([16, 32, 64]))
            vm.test_set_tiles(64, 0, blk)
            n = int(rng.integers(100, 8000))
            keys = _structured(rng, n, dtype)
            vals = np.arange(n, dtype=np.uint32) if trial % 3 else None
            nblocks = int(rng.integers(6, 40))
            bounded_vs_oracle(vm, keys, vals, scratch=nblocks * blk, minrun=int(rng.choice([0, 1, 4])))
    finally:
        vm.test_set_tiles(0, 0, 0)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_bounded_configs_reduced(vm, cfg):
    vm.test_set_tiles(0, 0, 0)
    n = 1 << 18
    k, v = W.make(cfg, n=n, device="cpu")
    st = bounded_vs_oracle(vm, W.to_numpy(k), None if v is None else W.to_numpy(v), scratch=cap(n))
    assert st["rounds"] > 0


def test_bounded_cfg2_full(vm):
    """cfg2 at its BASELINE.json size and cap: n = 2^24, scratch = 4 sqrt(n log2 n)
    = 80,264 elements; identical to the unbounded sort and to the oracle."""
    vm.test_set_tiles(0, 0, 0)
    vm.test_set_minrun(0)
    n = 1 << 24
    S = cap(n)
    assert S == 80264
    k, v = W.cfg2(device="cuda")
    k1, v1 = k.clone(), v.clone()
    st_b = vm.sort_(k, v, scratch=S, stats=True)
    st_u = vm.sort_(k1, v1, stats=True)
    torch.cuda.synchronize()
    assert torch.equal(k.view(torch.int32), k1.view(torch.int32))
    assert torch.equal(v.view(torch.int32), v1.view(torch.int32))
    assert st_b["scratch_bytes"] <= S * 8
    assert st_b["peak_extra_device_bytes"] < st_u["peak_extra_device_bytes"]


def test_bounded_budget_error(vm):
    vm.test_set_tiles(0, 0, 0)
    k = torch.randint(0, 1000, (100000,), dtype=torch.int32, device="cuda").view(torch.uint32)
    with pytest.raises(vm.VmpsError) as e:
        vm.sort_(k, scratch=60)  # fewer than 6 blocks of the minimum 16 elements
    assert e.value.status == 3


def _skip_input(rng, n, kind):
    """Inputs whose merges leave whole blocks in place: runs over disjoint,
    increasing value ranges (every merge a concatenation), and runs whose
    heads / tails do not overlap the neighbour (identity prefix / suffix
    tiles next to real merges)."""
    if kind == "concat":
        x = np.arange(n, dtype=np.int64) * 4
        cuts = np.sort(rng.integers(1, n, max(1, n // 300)))
        x[cuts] -= 1  # one descent per run: many runs, disjoint ranges
        return x.astype(np.uint32)
    x = np.empty(n, np.int64)
    cuts = np.concatenate([[0], np.sort(rng.integers(1, n, max(1, n // 500))), [n]])
    base = 0
    for a, b in zip(cuts[:-1], cuts[1:]):
        L = b - a
        # a run: a low prefix, a middle that overlaps the next run, a high suffix
        seg = np.sort(rng.integers(base, base + 3 * L, L))
        x[a:b] = seg
        base += L  # next run starts inside this run's range: partial overlap
    return x.astype(np.uint32)


@pytest.mark.parametrize("kind", ["concat", "overlap"])
def test_bounded_block_skip(vm, kind):
    """Clean blocks (every output already in place) are skipped -- zero bytes
    moved -- and the result still equals the oracle; concatenations need
    almost no rounds."""
    rng = np.random.default_rng(77 if kind == "concat" else 78)
    try:
        for trial in range(12):
            blk = int(rng.choice([16, 32, 64]))
            vm.test_set_tiles(64, 0, blk)
            n = int(rng.integers(2000, 20000))
            keys = _skip_input(rng, n, kind)
            vals = np.arange(n, dtype=np.uint32)
            st = bounded_vs_oracle(vm, keys, vals, scratch=int(rng.integers(6, 30)) * blk,
                                   minrun=int(rng.choice([1, 4])))
            if kind == "concat":
                assert st["rounds"] <= st["levels_executed"] + 2, st
    finally:
        vm.test_set_tiles(0, 0, 0)


def test_bounded_blocks_below_minrun(vm):
    """Blocks smaller than minrun at a size where the dirty-block scan (n/P + 1
    entries) is longer than the per-run arrays (n/minrun + 2): scratch = 200
    elements gives 16-element blocks at minrun 32 (the scan's
    temporary was sized by the run count and overflowed).  Identical to the
    oracle."""
    vm.test_set_tiles(0, 0, 0)
    n = 1 << 20
    k, v = W.cfg2(n=n, device="cpu")
    st = bounded_vs_oracle(vm, W.to_numpy(k), W.to_numpy(v), scratch=200)
    assert st["block_elems"] == 16 and st["minrun"] == 32


@pytest.mark.parametrize("chunk,n,dtype,kind", [(1 << 16, 1_000_003, np.uint32, "mixed"),
                                                (1 << 14, 300_000, np.uint64, "structured"),
                                                (1 << 15, 500_000, np.float32, "structured"),
                                                (1 << 12, 200_000, np.uint32, "longruns")])
def test_bounded_chunked(vm, chunk, n, dtype, kind):
    """The dyadic-cell scratch-bounded mode (n > 2 cells: runs grouped by the
    level-q dyadic cell of their midpoints, each cell's subtree sorted by the
    bounded engine with the global powers, Alg. 1 over the cell results):
    identical to the oracle's stable sort, with exactly the oracle's merge
    cost M and run count (the executed tree is the whole plan); element
    scratch within the cap; plan metadata sized by a cell, not by n."""
    rng = np.random.default_rng(chunk + n)
    if kind == "mixed":
        keys = W.to_numpy(W.cfg5(n=n, device="cpu")[0])
    elif kind == "longruns":  # runs much longer than a cell, ascending and strictly descending
        keys = np.empty(n, np.uint32)
        cuts = [0, 30_000, 90_000, 90_005, 150_000, n]
        for q, (a, b) in enumerate(zip(cuts[:-1], cuts[1:])):
            seg = np.sort(rng.integers(0, 1 << 31, b - a)).astype(np.uint32)
            keys[a:b] = seg[::-1] if q % 2 else seg
    else:
        keys = _structured(rng, n, dtype)
    vals = np.arange(n, dtype=np.uint32)
    S = cap(n)
    ko, vo, _, ost = oracle.sort(keys, vals)
    try:
        vm.test_set_bd_chunk(chunk)
        k = W.from_numpy(keys, "cuda")
        v = W.from_numpy(vals, "cuda")
        st = vm.sort_(k, v, scratch=S, stats=True)
        torch.cuda.synchronize()
        meta_chunked = st["metadata_bytes"]
    finally:
        vm.test_set_bd_chunk(0)
    assert W.to_numpy(k).view(np.uint8).tobytes() == ko.view(np.uint8).tobytes()
    assert (W.to_numpy(v) == vo).all()
    assert st["merge_cost_M"] == ost["merge_cost_M"] and st["runs"] == ost["runs"]
    w = keys.dtype.itemsize + 4
    assert st["scratch_bytes"] <= S * w
    st1 = vm.sort_(W.from_numpy(keys, "cuda"), W.from_numpy(vals, "cuda"), scratch=S, stats=True)
    assert meta_chunked < st1["metadata_bytes"]


@pytest.mark.parametrize("blk,n,dtype,hv,minrun", [(32, 150_001, np.float32, False, 0), (64, 200_000, np.uint64, True, 4),
                                                    (16, 70_003, np.uint32, True, 1), (16, 90_000, np.uint32, False, 0)])
def test_bounded_cells_small_blocks(vm, blk, n, dtype, hv, minrun):
    """Dyadic cells of 4096 elements over one shared block table whose
    blocks (16-64 elements, Z = 64) are far smaller than a cell: cell edges
    fall inside blocks, so the first block of most cells and detection
    chunks is brought home before it is read in place (bd_home); keys only
    and with payload, a partial last block; result, M and run count equal
    the oracle's."""
    rng = np.random.default_rng(blk * 1000 + n)
    keys = _structured(rng, n, dtype)
    vals = np.arange(n, dtype=np.uint32) if hv else None
    try:
        vm.test_set_tiles(64, 0, blk)
        vm.test_set_bd_chunk(4096)
        st = bounded_vs_oracle(vm, keys, vals, scratch=12 * blk, minrun=minrun)
        _, _, _, ost = oracle.sort(keys, vals, minrun_override=minrun)
        assert st["runs"] == ost["runs"]
    finally:
        vm.test_set_bd_chunk(0)
        vm.test_set_tiles(0, 0, 0)
        vm.test_set_minrun(0)


@pytest.mark.parametrize("nruns,n,dtype", [(2, 400_000, np.uint32), (5, 300_001, np.uint64), (9, 200_000, np.float32)])
def test_merge_runs_bounded(vm, nruns, n, dtype):
    """vmps_merge_runs_bounded (the multi-GPU bounded protocol's re-merge):
    adjacent sorted runs merged in place within the scratch cap, ties to the
    earlier run -- the stable sort of the concatenation (oracle)."""
    rng = np.random.default_rng(nruns * 7 + n)
    keys = _structured(rng, n, dtype)
    cuts = sorted(set(int(c) for c in rng.integers(1, n, nruns - 1)))
    starts = [0] + cuts
    for a, b in zip(starts, starts[1:] + [n]):  # sort each run (stable, by the key order)
        idx = np.argsort(R_image(keys[a:b]), kind="stable")
        keys[a:b] = keys[a:b][idx]
    vals = np.arange(n, dtype=np.uint32)
    ko, vo, _, _ = oracle.sort(keys, vals)
    k, v = W.from_numpy(keys, "cuda"), W.from_numpy(vals, "cuda")
    vm.merge_runs_bounded(k, v, starts, scratch=cap(n))
    torch.cuda.synchronize()
    assert W.to_numpy(k).view(np.uint8).tobytes() == ko.view(np.uint8).tobytes()
    assert (W.to_numpy(v) == vo).all()


def R_image(a):
    from tests.test_dist import image_np
    return image_np(a)
