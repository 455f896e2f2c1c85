"""GPU parity on the paper's own workload:
n ~ U[9 N/10, N] with N = 10^7 (general, non-power-of-two n: minrun 35-39),
integers uniform in [100, 10^9], pre-sorted runs of length Geom(1/S) for the
paper's S sweep.  `int`: keys + payload (= input index) and the merge plan,
both against the oracle, exactly.  Blobs (30 u32 words, lexicographic,
P:760-777) and `ptr` (the permutation): against oracle.sort_records byte for
byte at a reduced N, and at the paper's full N by properties that pin the
stable lexicographic sort completely (every output row >= its predecessor
lexicographically, the permutation is a permutation, equal records keep
their input order, records_out = records[perm])."""
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
    vm.test_set_tiles(0, 0, 0)
    return vm


@pytest.mark.parametrize("S", W.PAPER_S)
def test_paper_int_vs_oracle(vm, S):
    d, n = W.paper_input(S, "int", seed=0)
    assert 9 * 10 ** 6 <= n <= 10 ** 7
    kn = W.to_numpy(d)
    vn = np.arange(n, dtype=np.uint32)
    ko, vo, oplan, ost = oracle.sort(kn, vn)
    k, v = W.from_numpy(kn, "cuda"), W.from_numpy(vn, "cuda")
    st = vm.sort_(k, v, stats=True)
    torch.cuda.synchronize()
    assert st["minrun"] == ost["minrun"] == oracle.minrun(n)
    assert (W.to_numpy(k) == ko).all(), "keys differ"
    assert (W.to_numpy(v) == vo).all(), "payload (stability) differs"
    assert st["runs"] == ost["runs"] and st["merge_cost_M"] == ost["merge_cost_M"]
    p = vm.merge_plan(W.from_numpy(kn, "cuda"))
    assert (p.run_start.cpu().numpy() == oplan.run_start.astype(np.int64)).all()
    assert (p.run_kind.cpu().numpy() == oplan.run_kind).all()
    om = np.stack([oplan.merges[f].astype(np.int64) for f in ("i", "j", "k", "power")], axis=1)
    assert (p.merges.cpu().numpy() == om).all(), "merge plan differs"


@pytest.mark.parametrize("kind", ["randomBlob30", "zeroBlob30", "ptr"])
@pytest.mark.parametrize("S", [2, 10 ** 3, 10 ** 6])
def test_paper_blobs_vs_oracle(vm, kind, S):
    d, n = W.paper_input(S, "randomBlob30" if kind == "ptr" else kind, seed=1, N=200_000)
    recs = W.to_numpy(d).reshape(n, 30)
    want = oracle.sort_records(recs)
    r = torch.from_numpy(recs.view(np.int32)).cuda()
    out, pm = vm.sort_records(r, perm=True)
    torch.cuda.synchronize()
    assert (pm.cpu().numpy().astype(np.int64) == want).all(), "permutation differs"
    if kind != "ptr":
        assert out.cpu().numpy().view(np.uint32).tobytes() == recs[want].tobytes(), "records differ"


def _lex_sorted_stable(out: torch.Tensor, perm: torch.Tensor) -> bool:
    """Row r-1 <= row r lexicographically (u32 words, word 0 most
    significant) for every r, and equal rows in increasing input order."""
    a = out.to(torch.int64) & 0xFFFFFFFF
    diff = a[1:] != a[:-1]
    anyd = diff.any(dim=1)
    first = torch.argmax(diff.to(torch.int32), dim=1)  # first differing word (0 if equal)
    rows = torch.arange(a.shape[0] - 1, device=a.device)
    prev = a[:-1][rows, first]
    cur = a[1:][rows, first]
    pm = perm.to(torch.int64) & 0xFFFFFFFF
    return bool(((~anyd) | (cur > prev)).all()) and bool((anyd | (pm[1:] > pm[:-1])).all())


@pytest.mark.parametrize("kind", ["randomBlob30", "zeroBlob30"])
def test_paper_blobs_full_size(vm, kind):
    """The paper's N = 10^7 blobs: the output is the stable lexicographic sort,
    checked completely on the device."""
    d, n = W.paper_input(2, kind, seed=0, device="cuda")
    r = d.view(torch.int32).view(n, 30)
    out, pm = vm.sort_records(r, perm=True)
    torch.cuda.synchronize()
    p64 = pm.to(torch.int64) & 0xFFFFFFFF
    assert bool((torch.bincount(p64, minlength=n) == 1).all()), "not a permutation"
    assert torch.equal(out, r[p64]), "records_out != records[perm]"
    assert _lex_sorted_stable(out, pm), "not the stable lexicographic order"
