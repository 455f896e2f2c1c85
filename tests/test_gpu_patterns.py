"""GPU parity on structured inputs at ~2^20 (ragged n; among them skewed
key values -- powers of two, two far-apart clusters -- in sorted and
reversed segments): the default schedule
(two tree levels per HBM pass, 4-way merges) and one level per pass, both
leaf engines' default, against the CPU oracle, bit-exact (keys, payloads,
run count and merge cost)."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

N = (1 << 20) + 12345


def _patterns(n, rng):
    x = np.arange(n, dtype=np.uint64)
    yield "sorted", x.copy()
    yield "reverse", x[::-1].copy()
    h = n // 2
    yield "organ_pipe", np.concatenate([x[:h], x[:n - h][::-1]])
    for L in (33, 100, 5000):
        yield f"sawtooth{L}", (x % L)
    yield "all_equal", np.full(n, 7, np.uint64)
    yield "alternating", (x % 2)
    y = x.copy()
    sw = rng.integers(0, n, n // 100)
    y[sw], y[(sw + 1) % n] = y[(sw + 1) % n], y[sw]
    yield "nearly_sorted", y
    yield "desc_plateaus", np.repeat(np.arange(n // 64 + 1, dtype=np.uint64)[::-1], 64)[:n]
    r = rng.integers(0, 1 << 32, n, dtype=np.uint64)
    cuts = np.sort(rng.integers(0, n, 300))
    for a, b in zip(cuts[:-1:2], cuts[1::2]):
        r[a:b] = np.sort(r[a:b])[::-1] if (a & 1) else np.sort(r[a:b])
    yield "mixed_runs", r
    # skewed key values with sorted / reversed segments: huge gaps, heavy ties
    # and two far-apart clusters stress the partition's regula falsi probes
    # (interpolated positions, exact brackets) at every merge level
    def runs_of(v):
        cuts = np.sort(rng.integers(0, n, 400))
        for a, b in zip(cuts[:-1:2], cuts[1::2]):
            v[a:b] = np.sort(v[a:b])[::-1] if (a & 1) else np.sort(v[a:b])
        return v
    yield "pow2_skew", runs_of(np.left_shift(np.uint64(1), rng.integers(0, 64, n).astype(np.uint64)))
    lo = rng.integers(0, 1000, n).astype(np.uint64)
    yield "two_clusters", runs_of(np.where(rng.random(n) < 0.5, lo, np.uint64(0xFFFFFFFFFFFFFFFF) - lo))


@pytest.fixture(scope="module")
def vm():
    import paper_2605_27147_b200 as vm
    assert torch.cuda.is_available()
    vm.lib()
    yield vm
    vm.test_set_mode()
    vm.test_set_tiles(0, 0, 0)
    vm.test_set_minrun(0)


@pytest.mark.parametrize("levels", [2, 1])
@pytest.mark.parametrize("dtype", [np.uint32, np.uint64, np.float32])
def test_patterns_vs_oracle(vm, levels, dtype):
    rng = np.random.default_rng(700 + levels + (dtype == np.uint64) * 3 + (dtype == np.float32) * 5)
    vm.test_set_mode(levels)
    vm.test_set_tiles(0, 0, 0)
    vm.test_set_minrun(0)
    try:
        for name, base in _patterns(N, rng):
            if dtype == np.float32:
                keys = (base.astype(np.float64) - N / 2).astype(np.float32)
            else:
                keys = base.astype(dtype)
            vals = np.arange(N, dtype=np.uint32)
            ko, vo, _, ost = oracle.sort(keys, vals, variant=oracle.VARIANT_A)
            k = W.from_numpy(keys, "cuda")
            v = W.from_numpy(vals, "cuda")
            st = vm.sort_(k, v, stats=True)
            torch.cuda.synchronize()
            assert W.to_numpy(k).view(np.uint8).tobytes() == ko.view(np.uint8).tobytes(), name
            assert (W.to_numpy(v) == vo).all(), name
            assert st["runs"] == ost["runs"] and st["merge_cost_M"] == ost["merge_cost_M"], name
    finally:
        vm.test_set_mode()


@pytest.mark.parametrize("dtype", [np.uint32, np.uint64, np.float32])
def test_patterns_small_tiles_vs_oracle(vm, dtype):
    """The same patterns with 16-output merge tiles: ~65,000 tiles per level,
    so the large-level partition path runs (a thread per chain of hinted
    4-way splits with regula falsi steps) instead of the warp-per-tile one."""
    rng = np.random.default_rng(900 + (dtype == np.uint64) * 3 + (dtype == np.float32) * 5)
    vm.test_set_mode(2)
    vm.test_set_tiles(0, 16, 0)
    vm.test_set_minrun(0)
    try:
        for name, base in _patterns(N, rng):
            if dtype == np.float32:
                keys = (base.astype(np.float64) - N / 2).astype(np.float32)
            else:
                keys = base.astype(dtype)
            vals = np.arange(N, dtype=np.uint32)
            ko, vo, _, ost = oracle.sort(keys, vals, variant=oracle.VARIANT_A)
            k = W.from_numpy(keys, "cuda")
            v = W.from_numpy(vals, "cuda")
            st = vm.sort_(k, v, stats=True)
            torch.cuda.synchronize()
            assert W.to_numpy(k).view(np.uint8).tobytes() == ko.view(np.uint8).tobytes(), name
            assert (W.to_numpy(v) == vo).all(), name
            assert st["runs"] == ost["runs"] and st["merge_cost_M"] == ost["merge_cost_M"], name
    finally:
        vm.test_set_mode()
        vm.test_set_tiles(0, 0, 0)
