"""Randomised GPU cases (scripts/fuzz_gpu.py): sizes 0 .. 2^23, u32 / u64 /
f32 keys (f32 with +-0, +-inf and NaN payloads), keys-only and pairs, nine
input patterns, unbounded and scratch-bounded modes, one or two tree levels
per pass, and the minrun / fused-subtree / tile / block test hooks.  Each
case is compared bit-exact with the plain definition of the result, the
stable sort under the key order (numpy's stable argsort of the
order image), keys and payload (the input position)."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))


@pytest.mark.parametrize("seed", [101, 202, 303, 404])
def test_fuzz_against_definition(seed):
    import fuzz_gpu
    failed, skipped, _ = fuzz_gpu.run(40, seed)
    assert not failed, failed[:3]
    assert skipped <= 4


@pytest.mark.parametrize("seed", [11, 22, 33])
def test_fuzz_plan_against_oracle(seed):
    """The merge plan (run starts, kinds, Alg. 1's merges with powers, in
    order) of the fuzz patterns at n <= 2^18 and random minrun, against the
    oracle's plan (ExtractRun P:399/756, power P:445-446, Alg. 1)."""
    import numpy as np
    import oracle
    import paper_2605_27147_b200 as vm
    import fuzz_gpu
    import workloads as W
    rng = np.random.default_rng(seed)
    pats = ["uniform", "few", "equal", "segments", "segments_rev", "mixed", "sawtooth", "sorted", "reversed"]
    try:
        for _ in range(25):
            kt = str(rng.choice(["u32", "u64", "f32"]))
            n = int(np.exp(rng.uniform(np.log(2), np.log(1 << 18))))
            pat = str(rng.choice(pats))
            minrun = int(rng.choice([0, 0, 1, 3, 8, 32]))
            k0 = fuzz_gpu.gen(rng, n, kt, pat)
            vm.test_set_minrun(minrun)
            op, _ = oracle.plan(k0, minrun_override=minrun)
            p = vm.merge_plan(W.from_numpy(k0, "cuda"))
            case = (kt, n, pat, minrun)
            assert (p.run_start.cpu().numpy() == op.run_start.astype(np.int64)).all(), case
            assert (p.run_kind.cpu().numpy() == op.run_kind).all(), case
            got = [tuple(int(x) for x in row) for row in p.merges.cpu().numpy()]
            want = [(int(m["i"]), int(m["j"]), int(m["k"]), int(m["power"])) for m in op.merges]
            assert got == want, case
    finally:
        vm.test_set_minrun(0)


@pytest.mark.parametrize("seed", [7, 8])
def test_fuzz_host_buffers(seed):
    """The host-buffer entry points (vmps_sort_*_host: copy in, device sort,
    copy out, one stream), in place and out of place, pageable and pinned
    host memory, against the stable sort by definition."""
    import numpy as np
    import torch
    import paper_2605_27147_b200 as vm
    import fuzz_gpu
    rng = np.random.default_rng(seed)
    for _ in range(12):
        kt = str(rng.choice(["u32", "u64", "f32"]))
        n = int(np.exp(rng.uniform(0, np.log(1 << 21))))
        pat = str(rng.choice(["uniform", "few", "segments", "mixed", "sawtooth", "reversed"]))
        hv, pin, oop = bool(rng.random() < 0.7), bool(rng.random() < 0.5), bool(rng.random() < 0.5)
        k0 = fuzz_gpu.gen(rng, n, kt, pat)
        perm = np.argsort(fuzz_gpu.order_image(k0, kt), kind="stable")
        bits = k0.view(np.uint64) if kt == "u64" else k0.view(np.uint32)
        # f32 keys travel as a float32 tensor (an int32 one would be read as u32)
        kh = torch.from_numpy(k0.copy() if kt == "f32" else bits.view(np.int64 if kt == "u64" else np.int32).copy())
        vh = torch.arange(n, dtype=torch.int32) if hv else None
        if pin:
            kh = kh.pin_memory()
            vh = None if vh is None else vh.pin_memory()
        ko = torch.empty_like(kh) if oop else None
        vo = torch.empty_like(vh) if (oop and hv) else None
        vm.sort_host_(kh, vh, out_keys=ko, out_values=vo)
        torch.cuda.synchronize()
        rk = (ko if oop else kh).numpy().view(bits.dtype)  # bit patterns
        case = (kt, n, pat, hv, pin, oop)
        assert np.array_equal(rk, bits[perm]), case
        if hv:
            assert np.array_equal((vo if oop else vh).numpy().astype(np.int64), perm), case
        if oop:  # the input is left as it was
            assert np.array_equal(kh.numpy().view(bits.dtype), bits), case


@pytest.mark.parametrize("seed", [5, 6])
def test_fuzz_dist_virtual_ranks(seed):
    """The native multi-GPU sort (vmps_sort_*_dist: exact splitters, tie split
    in rank order, exchange, stable merge) on g = 2..6 virtual ranks with
    random shard sizes (empty shards, one non-empty shard) and the fuzz
    patterns (heavy ties included): the concatenated rank outputs are the
    stable sort of the concatenated shards by definition, and every rank
    keeps its element count."""
    import numpy as np
    import paper_2605_27147_b200 as vm
    import fuzz_gpu
    import workloads as W
    from tests import vranks
    rng = np.random.default_rng(seed)
    for _ in range(4):
        g = int(rng.integers(2, 7))
        kt = str(rng.choice(["u32", "u64", "f32"]))
        pat = str(rng.choice(["uniform", "few", "equal", "segments", "mixed", "sawtooth"]))
        r = rng.random()
        if r < 0.2:
            sizes = [0] * g
            sizes[int(rng.integers(0, g))] = int(rng.integers(1, 200_000))
        else:
            sizes = [int(rng.integers(0, 300_000)) if rng.random() < 0.8 else 0 for _ in range(g)]
        n = sum(sizes)
        k0 = fuzz_gpu.gen(rng, n, kt, pat)
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        ks = [k0[offs[q]:offs[q + 1]].copy() for q in range(g)]
        vs = [np.arange(offs[q], offs[q + 1], dtype=np.uint32) for q in range(g)]

        def fn(rank, comm):
            kd = W.from_numpy(ks[rank], "cuda")
            vd = W.from_numpy(vs[rank], "cuda")
            vm.sort_dist_native_(comm, kd, vd)
            return W.to_numpy(kd), W.to_numpy(vd)

        outs = vranks.run(g, fn)
        perm = np.argsort(fuzz_gpu.order_image(k0, kt), kind="stable")
        bits = k0.view(np.uint64) if kt == "u64" else k0.view(np.uint32)
        case = (g, kt, pat, sizes)
        for q in range(g):
            assert len(outs[q][0]) == sizes[q], case
        got = np.concatenate([o[0] for o in outs]).view(bits.dtype)
        assert np.array_equal(got, bits[perm]), case
        assert np.array_equal(np.concatenate([o[1] for o in outs]).astype(np.int64), perm), case


@pytest.mark.parametrize("seed", [9, 10])
def test_fuzz_records(seed):
    """vmps_sort_records on random record widths 1..33 words,
    with word values drawn from small alphabets (long tied prefixes, equal
    records) or the full range, against the stable lexicographic sort by
    definition (numpy lexsort: stable, word 0 most significant)."""
    import numpy as np
    import torch
    import paper_2605_27147_b200 as vm
    rng = np.random.default_rng(seed)
    for _ in range(10):
        words = int(rng.integers(1, 34))
        n = int(np.exp(rng.uniform(0, np.log(300_000))))
        alpha = int(rng.choice([1, 2, 3, 16, 2**32]))
        r = rng.integers(0, alpha, (n, words), dtype=np.uint64).astype(np.uint32)
        if rng.random() < 0.3 and n > 1:  # runs of equal records
            r = r[np.sort(rng.integers(0, n, n))]
        want = np.lexsort(r.T[::-1]) if n else np.zeros(0, np.int64)
        out, pm = vm.sort_records(torch.from_numpy(r.view(np.int32).copy()).cuda(), perm=True)
        torch.cuda.synchronize()
        case = (words, n, alpha)
        assert np.array_equal(pm.cpu().numpy().astype(np.int64), want), case
        assert out.cpu().numpy().view(np.uint32).tobytes() == r[want].tobytes(), case
