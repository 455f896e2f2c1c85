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
