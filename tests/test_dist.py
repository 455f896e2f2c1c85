"""Multi-GPU path: the sharded-sort protocol of
paper_2605_27147_b200/dist.py run by 2 and 3 gloo ranks on CPU (the compute
ops replaced by NumPy stand-ins defined here, test-side only), checked against
the oracle's stable sort of the concatenated shards; plus the splitter rule.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests import refcheck as R


def image_np(a: np.ndarray) -> np.ndarray:
    """Order image (test-side): u32/u64 as is; f32 per reading R5."""
    if a.dtype == np.float32:
        b = a.view(np.uint32).astype(np.uint64)
        nan = (b & 0x7FFFFFFF) > 0x7F800000
        img = np.where(b >> 31, b ^ 0xFFFFFFFF, b | 0x80000000)
        return np.where(nan, np.uint64(0xFFFFFFFF), img).astype(np.uint64)
    return a.astype(np.uint64)


def _np(t):
    import workloads as W
    return W.to_numpy(t)


class NumpyOps:
    """CPU stand-ins for the three data-path operations."""

    def local_sort(self, keys, vals):
        import workloads as W
        a = _np(keys)
        idx = np.argsort(image_np(a), kind="stable")
        keys.copy_(W.from_numpy(a[idx]))
        if vals is not None:
            v = _np(vals)
            vals.copy_(W.from_numpy(v[idx]))

    def count(self, keys, probes):
        img = image_np(_np(keys))
        p = np.array(probes, dtype=np.uint64)
        lt = np.searchsorted(img, p, side="left").astype(np.int64)
        le = np.searchsorted(img, p, side="right").astype(np.int64)
        return torch.from_numpy(lt), torch.from_numpy(le)

    def merge_runs(self, keys, vals, starts):
        self.local_sort(keys, vals)  # stable sort of concatenated sorted pieces == stable merge


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shards, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import workloads as W
    from paper_2605_27147_b200.dist import sort_dist
    k, v = shards[rank]
    res = sort_dist(W.from_numpy(k), W.from_numpy(v), ops=NumpyOps())
    out_q.put((rank, _np(res.keys), _np(res.vals), res.send_counts, res.recv_counts, res.rounds))
    dist.destroy_process_group()


def _run(world, shards):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shards, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(outs, key=lambda x: x[0])


@pytest.mark.parametrize("world,dtype,sizes", [
    (2, np.uint32, [3000, 3000]),
    (2, np.uint64, [2500, 2500]),
    (2, np.float32, [2000, 2000]),
    (3, np.uint32, [1000, 2500, 1700]),   # unequal shards
])
def test_sort_dist_gloo(world, dtype, sizes):
    rng = np.random.default_rng(world * 100 + len(sizes))
    shards, allk = [], []
    base = 0
    for n in sizes:
        if dtype == np.float32:
            k = rng.choice(np.array([0.0, -0.0, 1.5, -2.0, np.nan, 3.0], np.float32), n)
        elif dtype == np.uint64:
            k = rng.integers(0, 5, n).astype(np.uint64) << np.uint64(40)
        else:
            k = rng.integers(0, 7, n).astype(np.uint32)  # heavy ties across shards
        v = np.arange(base, base + n, dtype=np.uint32)
        shards.append((k, v))
        allk.append(k)
        base += n
    outs = _run(world, shards)
    gk = np.concatenate([o[1] for o in outs])
    gv = np.concatenate([o[2] for o in outs])
    ek, ev = R.stable_sorted(np.concatenate(allk))
    assert gk.view(np.uint8).tobytes() == ek.view(np.uint8).tobytes()
    assert (gv == ev).all()
    # rank p holds global output ranks [R_p, R_{p+1}) with R_t = t N / g
    N = sum(sizes)
    for p, o in enumerate(outs):
        assert len(o[1]) == (p + 1) * N // world - p * N // world


def test_split_points_rule():
    from paper_2605_27147_b200.dist import split_points
    # ranks 0..2 with lt/le counts at v*: the tie group is taken in rank order
    assert split_points(10, [3, 2, 1], [6, 6, 4]) == [6, 3, 1]   # need 4 of the ties: 3 from r0, 1 from r1
    assert split_points(6, [3, 2, 1], [6, 6, 4]) == [3, 2, 1]    # no ties taken
    assert split_points(16, [3, 2, 1], [6, 6, 4]) == [6, 6, 4]   # all ties taken
