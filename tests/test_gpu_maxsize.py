"""Maximum sizes: the largest array the ABI accepts (VMPS_MAX_N = 2^32 - 2^16,
the next size rejected) and a size
past 2^31 (where a signed 32-bit position would overflow), checked by exact
properties that determine a stable sort uniquely at any size: keys
non-decreasing under the key order, the payload (= input position) a
permutation, increasing within every run of equal keys; for keys only,
non-decreasing plus an unchanged multiset fingerprint (high-16-bit
histogram and a nonlinear mix sum).  Inputs mix unsorted,
sorted and strictly descending segments (every run kind) and are built chunk
by chunk on the device."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _fill(n, seed, dev):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    k = torch.empty(n, dtype=torch.int32, device=dev)
    C = 1 << 26
    for i, a in enumerate(range(0, n, C)):
        b = min(n, a + C)
        x = torch.randint(-(1 << 31), 1 << 31, (b - a,), generator=g, device=dev, dtype=torch.int64)
        if i % 3 == 1:
            x = torch.sort(x).values            # one long ascending run
        elif i % 3 == 2:
            x = torch.sort(x, descending=True).values  # strictly descending (w.h.p.): reversed in place
            x[: (b - a) // 2] = x[: (b - a) // 2] % 7   # plus a stretch of heavy ties
        k[a:b] = x.to(torch.int32)
    return k.view(torch.uint32)


def _img(k):
    return k.view(torch.int32).to(torch.int64) & 0xFFFFFFFF


def _check_sorted(k, C=1 << 27):
    n = k.numel()
    for a in range(0, n - 1, C):
        b = min(n, a + C + 1)
        seg = _img(k[a:b])
        assert bool((seg[1:] >= seg[:-1]).all()), f"not sorted near {a}"


def test_sort_pairs_past_2_31():
    import paper_2605_27147_b200 as vm
    dev = torch.device("cuda")
    n = (1 << 31) + 12345
    k = _fill(n, 31, dev)
    v = torch.arange(n, device=dev, dtype=torch.int64).to(torch.int32).view(torch.uint32)
    k0 = k.clone()
    st = vm.sort_(k, v, stats=True)
    torch.cuda.synchronize()
    assert st["n"] == n
    _check_sorted(k)
    # payload: a permutation of 0..n-1 and, within equal keys, increasing; key = k0[payload]
    C = 1 << 27
    seen = torch.zeros(n, dtype=torch.uint8, device=dev)
    for a in range(0, n, C):
        b = min(n, a + C)
        p = _img(v[a:b])
        seen[p] = 1
        assert bool((k0.view(torch.int32)[p] == k[a:b].view(torch.int32)).all()), "payload does not point at its key"
    assert int(seen.sum()) == n, "payload is not a permutation"
    for a in range(0, n - 1, C):
        b = min(n, a + C + 1)
        kk, pp = _img(k[a:b]), _img(v[a:b])
        eq = kk[1:] == kk[:-1]
        assert bool((pp[1:][eq] > pp[:-1][eq]).all()), "equal keys out of input order"
    del k, v, k0, seen


def _fingerprint(k, C=1 << 27):
    """Multiset fingerprint: the 65,536-bin histogram of the keys' high 16 bits
    plus a wrapped int64 sum of a nonlinear mix of every key -- a dropped,
    duplicated or altered key changes one of them (w.h.p. for the mix)."""
    n = k.numel()
    hist = torch.zeros(1 << 16, dtype=torch.int64, device=k.device)
    mix = torch.zeros((), dtype=torch.int64, device=k.device)
    for a in range(0, n, C):
        x = _img(k[a:min(n, a + C)])
        hist += torch.bincount(x >> 16, minlength=1 << 16)
        y = (x * 40503) ^ (x >> 7)
        y = y * 2654435761 + (y >> 13) * 97
        mix += y.sum()
    return hist, int(mix.item())


def test_sort_keys_max_n():
    import paper_2605_27147_b200 as vm
    dev = torch.device("cuda")
    n = (1 << 32) - (1 << 16)  # VMPS_MAX_N
    k = _fill(n, 32, dev)
    h0, m0 = _fingerprint(k)
    vm.sort_(k)
    torch.cuda.synchronize()
    _check_sorted(k)
    h1, m1 = _fingerprint(k)
    assert bool(torch.equal(h0, h1)), "multiset changed (high-16-bit histogram)"
    assert m0 == m1, "multiset changed (mix sum)"
    del k


def test_max_n_limit():
    import ctypes
    import paper_2605_27147_b200 as vm
    nb = ctypes.c_size_t(0)
    L = vm.lib()
    assert L.vmps_workspace_bytes((1 << 32) - (1 << 16), vm.KEY_U32, 0, -1, ctypes.byref(nb)) == vm.OK
    assert L.vmps_workspace_bytes((1 << 32) - (1 << 16) + 1, vm.KEY_U32, 0, -1, ctypes.byref(nb)) == vm.ERR_INVALID_ARG
