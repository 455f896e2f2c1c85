"""GPU parity of vmps_sort_records (the paper's blob types,
P:760-777) vs oracle.sort_records (stable lexicographic order): the
permutation exactly, and the gathered records byte for byte.  Cases: the
paper's randomBlob30 (words uniform in [100, 1e9]) and zeroBlob30 (only the
last word nonzero), ties on the leading pair (the LSD path), odd word counts,
one- and two-word records, the `ptr` form (permutation only), n = 1."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _check(recs_np, perm_only=False):
    import paper_2605_27147_b200 as vm
    r = torch.from_numpy(recs_np.view(np.int32)).cuda()
    want = oracle.sort_records(recs_np)
    if perm_only:
        _, pm = vm.sort_records(r, perm=True)
        torch.cuda.synchronize()
        assert (pm.cpu().numpy().astype(np.int64) == want).all()
        return
    out, pm = vm.sort_records(r, perm=True)
    torch.cuda.synchronize()
    assert (pm.cpu().numpy().astype(np.int64) == want).all(), "permutation differs"
    assert out.cpu().numpy().view(np.uint32).tobytes() == recs_np[want].tobytes(), "records differ"


@pytest.mark.parametrize("kind", ["randomBlob30", "zeroBlob30", "tiedLead", "ptr"])
def test_blob30(kind):
    rng = np.random.default_rng(7)
    n = 20_000
    if kind == "zeroBlob30":
        r = np.zeros((n, 30), np.uint32)
        r[:, 29] = rng.integers(100, 10 ** 9, n)
    else:
        r = rng.integers(100, 10 ** 9, (n, 30)).astype(np.uint32)
    if kind == "tiedLead":
        r[:, 0] = rng.integers(0, 3, n)
        r[:, 1] = rng.integers(0, 2, n)
        r[:, 2] = rng.integers(0, 5, n)
        r[::7] = r[0]  # fully equal records keep their input order
    _check(r, perm_only=(kind == "ptr"))


def test_constant_leading_pairs():
    """Pairs 0-1 equal in every record, pair 2 decides with ties, later pairs
    vary (the LSD path over the non-constant pairs only)."""
    rng = np.random.default_rng(9)
    n = 8000
    r = np.zeros((n, 9), np.uint32)
    r[:, 0] = 7
    r[:, 4] = rng.integers(0, 4, n)
    r[:, 5] = rng.integers(0, 2, n)
    r[:, 7] = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    r[::11, 7] = 3
    _check(r)
    all_equal = np.tile(np.array([[1, 2, 3]], np.uint32), (500, 1))
    _check(all_equal)


@pytest.mark.parametrize("words", [1, 2, 3, 5])
def test_word_counts(words):
    rng = np.random.default_rng(words)
    r = rng.integers(0, 4, (5001, words)).astype(np.uint32)
    r[:, -1] = rng.integers(0, 1 << 32, 5001, dtype=np.uint64).astype(np.uint32)
    _check(r)


def test_single_and_errors():
    import paper_2605_27147_b200 as vm
    _check(np.array([[5, 6, 7]], np.uint32))
    r = torch.zeros((4, 2), dtype=torch.int32, device="cuda")
    L = vm.lib()
    assert L.vmps_sort_records(r.data_ptr(), r.data_ptr(), None, 4, 2, None, 0, None) == vm.ERR_INVALID_ARG
    out = torch.empty_like(r)
    assert L.vmps_sort_records(r.data_ptr(), out.data_ptr(), None, 4, 2, None, 0, None) == vm.ERR_BUDGET
