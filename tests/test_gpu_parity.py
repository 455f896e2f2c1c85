"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, exact.

Keys, payloads and merge plans are compared element by element (bit-exact:
this is integer/byte/index work; f32 keys are compared as bit patterns).
Small cases cover many tiles, ragged tails, every key type and the
degenerate inputs; full-size BASELINE.json configs are checked with exact
properties that determine a stable sort uniquely (sorted under the key order,
payload = original index strictly increasing within equal keys, payload a
permutation) plus the oracle's plan-only pass (run starts, kinds, merges).
"""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
from tests import refcheck as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vm():
    import paper_2605_27147_b200 as vm
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    vm.lib()
    yield vm
    vm.test_set_minrun(0)
    vm.test_set_tiles(0, 0, 0)


def _plan_tuples(merges_np):
    return [tuple(int(m[f]) for f in ("i", "j", "k", "power")) for m in merges_np]


def gpu_sort(vm, keys_np, vals_np):
    k = W.from_numpy(keys_np, "cuda")
    v = None if vals_np is None else W.from_numpy(vals_np, "cuda")
    st = vm.sort_(k, v, stats=True)
    torch.cuda.synchronize()
    return W.to_numpy(k), (None if v is None else W.to_numpy(v)), st


def check_case(vm, keys_np, vals_np, minrun=0, plan=True):
    vm.test_set_minrun(minrun)
    ko, vo, oplan, ost = oracle.sort(keys_np, vals_np, variant=oracle.VARIANT_A,
                                     minrun_override=minrun)
    gk, gv, gst = gpu_sort(vm, keys_np, vals_np)
    assert gk.view(np.uint8).tobytes() == ko.view(np.uint8).tobytes(), "keys differ"
    if vals_np is not None:
        assert (gv == vo).all(), "payload differs"
    assert gst["runs"] == ost["runs"]
    assert gst["merge_cost_M"] == ost["merge_cost_M"]
    if plan and len(keys_np) > 1:
        p = vm.merge_plan(W.from_numpy(keys_np, "cuda"))
        rs = p.run_start.cpu().numpy()
        assert (rs == oplan.run_start.astype(np.int64)).all(), "run starts differ"
        assert (p.run_kind.cpu().numpy() == oplan.run_kind).all(), "run kinds differ"
        got = [tuple(int(x) for x in row) for row in p.merges.cpu().numpy()]
        assert got == _plan_tuples(oplan.merges), "merge plan differs"


def _structured(rng, n, dtype):
    kind = int(rng.integers(0, 6))
    if dtype == np.float32:
        pool = np.array([0.0, -0.0, 1.0, -1.0, np.nan, np.inf, -np.inf, 2.5, -2.5, 1e-30],
                        np.float32)
        if kind < 3:
            x = pool[rng.integers(0, len(pool), n)]
        else:
            x = rng.standard_normal(n).astype(np.float32)
            cuts = np.sort(rng.integers(0, n + 1, max(1, n // 100)))
            for a, b in zip(cuts[:-1], cuts[1:]):
                x[a:b] = np.sort(x[a:b])[::-1] if rng.random() < 0.3 else np.sort(x[a:b])
            x[rng.random(n) < 0.01] = -0.0
            x[rng.random(n) < 0.01] = np.nan
        bits = x.view(np.uint32).copy()
        m = rng.random(n) < 0.02
        bits[m] = np.uint32(0xFFC00000) | rng.integers(0, 1 << 20, int(m.sum())).astype(np.uint32)
        return bits.view(np.float32)
    hi = (1 << 63) if dtype == np.uint64 else (1 << 32)
    if kind == 0:
        x = rng.integers(0, 8, n, dtype=np.uint64)
    elif kind == 1:
        x = rng.integers(0, hi, n, dtype=np.uint64)
    elif kind == 2:
        x = rng.integers(0, 1000, n, dtype=np.uint64)
        cuts = np.sort(rng.integers(0, n + 1, max(1, n // 50)))
        for a, b in zip(cuts[:-1], cuts[1:]):
            seg = np.sort(x[a:b])
            x[a:b] = seg[::-1] if rng.random() < 0.3 else seg
    elif kind == 3:
        x = np.arange(n, dtype=np.uint64)[::-1].copy()
        x[rng.integers(0, max(n, 1), max(1, n // 100))] = 5
    elif kind == 4:
        x = np.sort(rng.integers(0, 100, n, dtype=np.uint64))
    else:
        x = rng.integers(0, hi, n, dtype=np.uint64)
        x[: n // 2] = np.sort(x[: n // 2])
    return x.astype(dtype)


@pytest.mark.parametrize("dtype", [np.uint32, np.uint64, np.float32])
@pytest.mark.parametrize("with_vals", [False, True])
def test_random_small_default_tiles(vm, dtype, with_vals):
    rng = np.random.default_rng(100 + (dtype == np.uint64) * 7 + (dtype == np.float32) * 13)
    vm.test_set_tiles(0, 0, 0)
    for trial in range(25):
        n = int(rng.choice([2, 3, 63, 64, 65, 100, 1000, 4095, 4096, 4097, 9000, 20000, 70001]))
        keys = _structured(rng, n, dtype)
        vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32) if with_vals else None
        check_case(vm, keys, vals, minrun=int(rng.choice([0, 1, 2, 7, 32])))


@pytest.mark.parametrize("levels,leaf_radix", [(2, False), (1, False), (2, True)])
@pytest.mark.parametrize("dtype", [np.uint32, np.uint64, np.float32])
def test_random_small_tiny_tiles(vm, dtype, levels, leaf_radix):
    """Z = 64 and 16-element merge tiles: small inputs cross every level path;
    both merge schedules (1 or 2 tree levels per pass) and both leaf engines
    (a leaf batch then holds ~70 units and spans long leaves' gaps)."""
    rng = np.random.default_rng(200 + (dtype == np.uint64) + 2 * (dtype == np.float32))
    try:
        vm.test_set_mode(levels)
        vm.test_set_leaf(leaf_radix)
        vm.test_set_tiles(64, 16, 0)
        for trial in range(40):
            n = int(rng.integers(2, 6000))
            keys = _structured(rng, n, dtype)
            vals = np.arange(n, dtype=np.uint32)
            check_case(vm, keys, vals, minrun=int(rng.choice([0, 1, 2, 3, 16])))
    finally:
        vm.test_set_tiles(0, 0, 0)
        vm.test_set_mode()
        vm.test_set_leaf(False)


def test_edge_cases(vm):
    vm.test_set_tiles(0, 0, 0)
    cases = [
        np.zeros(0, np.uint32), np.zeros(1, np.uint32), np.array([2, 1], np.uint32),
        np.full(100000, 7, np.uint32),                      # all equal: one run
        np.arange(200000, dtype=np.uint32)[::-1].copy(),    # one strictly descending run
        np.arange(200000, dtype=np.uint32),                 # sorted: one long ascending run
        np.repeat(np.arange(1000, dtype=np.uint32)[::-1], 100),  # descending plateaus
        np.tile(np.array([3, 2, 1], np.uint32), 33333),
    ]
    for keys in cases:
        n = len(keys)
        vals = np.arange(n, dtype=np.uint32)
        if n <= 1:
            gk, gv, st = gpu_sort(vm, keys, vals) if n == 1 else (keys, vals, None)
            assert (gk == keys).all()
            continue
        check_case(vm, keys, vals)


@pytest.mark.parametrize("levels,leaf_radix", [(2, False), (1, False), (2, True)])
@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_configs_reduced_size_vs_oracle(vm, cfg, levels, leaf_radix):
    """Each BASELINE.json config shape at 2^18 (many merge levels), full oracle
    compare, both merge schedules and both leaf engines."""
    vm.test_set_tiles(0, 0, 0)
    vm.test_set_mode(levels)
    vm.test_set_leaf(leaf_radix)
    try:
        k, v = W.make(cfg, n=1 << 18, device="cpu")
        check_case(vm, W.to_numpy(k), None if v is None else W.to_numpy(v))
    finally:
        vm.test_set_mode()
        vm.test_set_leaf(False)


def _ord_image(k: torch.Tensor) -> torch.Tensor:
    """Order image for verification only (int64 for u32/f32; u64 split)."""
    if k.dtype == torch.float32:
        b = k.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        nan = (b & 0x7FFFFFFF) > 0x7F800000
        img = torch.where((b >> 31) == 1, b ^ 0xFFFFFFFF, b ^ 0x80000000)
        return torch.where(nan, torch.full_like(img, 0xFFFFFFFF), img)
    if k.dtype == torch.uint32:
        return k.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    return k.view(torch.int64) ^ (-(1 << 63))  # u64 -> signed order


def verify_stable_sorted(keys_in, vals_in, keys_out, vals_out):
    """Exact check that (keys_out, vals_out) is the stable sort of the input."""
    a = _ord_image(keys_out)
    assert bool((a[1:] >= a[:-1]).all()), "not sorted"
    if vals_in is not None:
        # payload = original index: strictly increasing within equal keys, and a permutation
        pv = vals_out.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        eq = a[1:] == a[:-1]
        assert bool(((pv[1:] > pv[:-1]) | ~eq).all()), "not stable"
        seen = torch.zeros(pv.numel(), dtype=torch.bool, device=pv.device)
        seen[pv] = True
        assert bool(seen.all()), "payload is not a permutation"
        src = _ord_image(keys_in)
        assert bool((src[pv] == a).all()), "keys do not travel with their payload"
        if keys_in.dtype == torch.float32:
            kb = keys_in.view(torch.int32)
            assert bool((kb[pv] == keys_out.view(torch.int32)).all())
    else:
        # keys only: output = input multiset in sorted order (bit patterns)
        bi = keys_in.view(torch.int32 if keys_in.element_size() == 4 else torch.int64)
        bo = keys_out.view(bi.dtype)
        assert bool((torch.sort(bi).values == torch.sort(bo).values).all()), "not a permutation"
        if keys_in.dtype == torch.float32:
            # -0.0 before +0.0 and NaN last are inside the order image; equal
            # images have equal bit patterns except NaNs (none in cfg4)
            pass


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_configs_full_size(vm, cfg):
    """BASELINE.json configs at full single-GPU size, in the bench's launch
    configuration: exact stable-sort properties + the oracle's plan."""
    vm.test_set_tiles(0, 0, 0)
    vm.test_set_minrun(0)
    k, v = W.make(cfg, device="cuda")
    k0 = k.clone()
    v0 = None if v is None else v.clone()
    st = vm.sort_(k, v, stats=True)
    torch.cuda.synchronize()
    verify_stable_sorted(k0, v0, k, v)
    # plan: oracle plan-only pass over the same keys
    oplan, ost = oracle.plan(W.to_numpy(k0))
    assert st["runs"] == ost["runs"]
    assert st["merge_cost_M"] == ost["merge_cost_M"]
    p = vm.merge_plan(k0)
    assert (p.run_start.cpu().numpy() == oplan.run_start.astype(np.int64)).all()
    assert (p.run_kind.cpu().numpy() == oplan.run_kind).all()
    om = np.stack([oplan.merges["i"], oplan.merges["j"], oplan.merges["k"],
                   oplan.merges["power"]], axis=1).astype(np.int64)
    assert (p.merges.cpu().numpy() == om).all()
    if cfg <= 2:  # the oracle's full sort is fast here: element-by-element compare
        ko, vo, _, _ = oracle.sort(W.to_numpy(k0), None if v0 is None else W.to_numpy(v0))
        assert (W.to_numpy(k) == ko).all()
        if v is not None:
            assert (W.to_numpy(v) == vo).all()


def test_workspace_and_errors(vm):
    import ctypes
    L = vm.lib()
    nb = vm.workspace_bytes(1 << 20, vm.KEY_U32, 1)
    assert nb > 8 * (1 << 20)
    k = torch.zeros(1000, dtype=torch.int32, device="cuda").view(torch.uint32)
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    rc = L.vmps_sort_keys(k.data_ptr(), 1000, 0, -1, ws.data_ptr(), 16, None, None)
    assert rc == 3  # VMPS_ERR_BUDGET
    rc = L.vmps_sort_keys(k.data_ptr() + 4, 999, 0, -1, ws.data_ptr(), 16, None, None)
    assert rc == 1  # misaligned
    rc = L.vmps_sort_keys(k.data_ptr(), 1000, 9, -1, ws.data_ptr(), 16, None, None)
    assert rc == 1  # bad key type


@pytest.mark.parametrize("dtype", [np.uint32, np.uint64, np.float32])
def test_host_entry_points(vm, dtype):
    """vmps_sort_*_host: host in -> device sort -> host out (in place and out of
    place, keys only and pairs), exact vs the oracle."""
    vm.test_set_tiles(0, 0, 0)
    vm.test_set_minrun(0)
    rng = np.random.default_rng(500 + (dtype == np.uint64) + 2 * (dtype == np.float32))
    for n in (1, 2, 5000, 70001):
        keys = _structured(rng, n, dtype)
        vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        ko, vo, _, _ = oracle.sort(keys, vals, variant=oracle.VARIANT_A)
        kk, _, _, _ = oracle.sort(keys, None, variant=oracle.VARIANT_A)
        hk = W.from_numpy(keys, "cpu").pin_memory()
        hv = W.from_numpy(vals, "cpu").pin_memory()
        outk, outv = torch.empty_like(hk).pin_memory(), torch.empty_like(hv).pin_memory()
        s = torch.cuda.Stream()
        vm.sort_host_(hk, hv, out_keys=outk, out_values=outv, stream=s)   # out of place
        s.synchronize()
        assert W.to_numpy(outk).view(np.uint8).tobytes() == ko.view(np.uint8).tobytes()
        assert (W.to_numpy(outv) == vo).all()
        assert W.to_numpy(hk).view(np.uint8).tobytes() == keys.view(np.uint8).tobytes()  # input untouched
        hk2 = W.from_numpy(keys, "cpu").pin_memory()
        vm.sort_host_(hk2)                                                 # keys only, in place
        torch.cuda.synchronize()
        assert W.to_numpy(hk2).view(np.uint8).tobytes() == kk.view(np.uint8).tobytes()


def test_concurrent_streams(vm):
    """Independent sorts on different streams with their own workspaces run
    concurrently (the ABI's thread-safety convention): each equals the oracle."""
    rng = np.random.default_rng(55)
    cases = []
    for dt in (np.uint32, np.uint64, np.float32, np.uint32):
        n = int(rng.integers(200_000, 600_000))
        k = _structured(rng, n, dt)
        v = np.arange(n, dtype=np.uint32)
        cases.append((k, v))
    streams = [torch.cuda.Stream() for _ in cases]
    wss = [vm.Workspace() for _ in cases]
    dev = [(W.from_numpy(k, "cuda"), W.from_numpy(v, "cuda")) for k, v in cases]
    torch.cuda.synchronize()
    for (dk, dv), s, ws in zip(dev, streams, wss):
        with torch.cuda.stream(s):
            vm.sort_(dk, dv, workspace=ws)
    torch.cuda.synchronize()
    for (k, v), (dk, dv) in zip(cases, dev):
        ko, vo, _, _ = oracle.sort(k, v)
        assert W.to_numpy(dk).view(np.uint8).tobytes() == ko.view(np.uint8).tobytes()
        assert (W.to_numpy(dv) == vo).all()
