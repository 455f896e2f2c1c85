"""CPU checks of bench.py's host-side verification helpers (the order image
used for the sortedness check, the multiset hash and the plan hash) against
plain NumPy / Python definitions, and of the reference arm's JSON line."""
import json
import os
import subprocess
import sys

import numpy as np
import torch

import bench
import workloads as W
from tests.test_dist import image_np


def test_order_image_matches_definition():
    rng = np.random.default_rng(1)
    f = rng.standard_normal(1000).astype(np.float32)
    f[:10] = [0.0, -0.0, np.nan, -np.nan, np.inf, -np.inf, 1e-38, -1e-38, 3.0, -3.0]
    got = bench.order_image(W.from_numpy(f)).numpy()
    assert (got.astype(np.uint64) == image_np(f)).all()
    u = rng.integers(0, 1 << 32, 1000, dtype=np.uint64).astype(np.uint32)
    assert (bench.order_image(W.from_numpy(u)).numpy().astype(np.uint64) == u.astype(np.uint64)).all()
    v = rng.integers(0, 1 << 63, 1000, dtype=np.uint64) | (rng.integers(0, 2, 1000, dtype=np.uint64) << np.uint64(63))
    img = bench.order_image(W.from_numpy(v)).numpy()
    # signed order of the image == unsigned order of the keys
    assert (np.argsort(img, kind="stable") == np.argsort(v, kind="stable")).all()


def test_mix_hash_is_a_multiset_hash():
    rng = np.random.default_rng(2)
    k = W.from_numpy(rng.integers(0, 1 << 32, 5000, dtype=np.uint64).astype(np.uint32))
    v = W.from_numpy(np.arange(5000, dtype=np.uint32))
    h = bench.mix_hash(k, v)
    p = torch.randperm(5000)
    assert bench.mix_hash(k[p].contiguous(), v[p].contiguous()) == h          # order does not matter
    kn = W.to_numpy(k).copy()
    kn[7] = kn[8]
    assert bench.mix_hash(W.from_numpy(kn), v) != h                            # a changed pair does
    vn = W.to_numpy(v).copy()
    vn[[3, 4]] = vn[[4, 3]]
    assert bench.mix_hash(k, W.from_numpy(vn)) != h                            # keys must travel with payloads


def test_plan_hash_distinguishes_records():
    i = torch.tensor([0, 0, 4]); j = torch.tensor([2, 4, 6]); k = torch.tensor([4, 8, 8])
    pw = torch.tensor([2, 1, 2]); od = torch.arange(3)
    h = bench.plan_hash_of(i, j, k, pw, od)
    assert bench.plan_hash_of(i, j, k, pw, od.flip(0)) != h
    assert bench.plan_hash_of(i, j, k, torch.tensor([2, 2, 2]), od) != h


def test_reference_arm_line():
    """--impl reference prints one JSON line with the contract's keys (tiny sample)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--ref-sample-log2", "14"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "cpu_baseline", "e2e", "config", "higher_is_better"):
        assert key in d
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "oracle"


def test_launcher_two_ranks():
    """`bench.py --gpus 2` outside torchrun spawns two ranks that join one gloo
    group (the launcher's rendezvous plumbing, no GPU); rank 0 reports n_gpus = 2."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--launcher-selftest"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d == {"launcher_selftest": True, "n_gpus": 2}
