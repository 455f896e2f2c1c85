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


# ---- distributed merge plan (dist.merge_plan_dist) -------------------------

class PlanFake:
    """CPU stand-ins for the plan's data-path operations, test-side: they know
    the global array, check the edge keys the protocol hands them (previous
    key, halo, n_end, minrun) and answer from the oracle's plan of the whole
    array.  The transfer table is a stand-in (entry s -> s + 1 mod 3 minrun,
    with the shard's true run count), so the composed entry states are checked
    too."""

    def __init__(self, glob):
        import oracle
        self.g = glob
        self.N = len(glob)
        self.oplan, _ = oracle.plan(glob)
        self.starts = self.oplan.run_start.astype(np.int64)
        self.mr = oracle.minrun(self.N)

    def _check_edges(self, keys, minrun, n_end, prev, halo):
        from paper_2605_27147_b200.dist import halo_len
        off = self.N - n_end
        n = keys.numel()
        assert minrun == self.mr
        assert (_np(keys).view(np.uint8) == self.g[off:off + n].view(np.uint8)).all()
        if off == 0:
            assert prev is None
        else:
            assert _np(prev).view(np.uint8).tobytes() == self.g[off - 1:off].view(np.uint8).tobytes()
        want = self.g[off + n: off + n + halo_len(minrun)]
        got = np.zeros(0, self.g.dtype) if halo is None else _np(halo)
        assert got.view(np.uint8).tobytes() == want.view(np.uint8).tobytes()
        return off, n

    def _mine(self, off, n):
        return np.nonzero((self.starts >= off) & (self.starts < off + n))[0]

    def chain(self, keys, minrun, n_end, prev, halo):
        off, n = self._check_edges(keys, minrun, n_end, prev, halo)
        c = len(self._mine(off, n))
        ns = 3 * minrun
        return torch.tensor([(((s + 1) % ns) << 32) | c for s in range(ns)], dtype=torch.int64)

    def runs(self, keys, minrun, n_end, prev, halo, entry, count, offset, out_starts):
        off, n = self._check_edges(keys, minrun, n_end, prev, halo)
        assert offset == off
        nonempty_before = len({int(np.searchsorted(np.cumsum(self.sizes), x, side="right"))
                               for x in range(off)}) if off else 0
        assert entry == nonempty_before % (3 * minrun)
        idx = self._mine(off, n)
        assert count == len(idx)
        out_starts.copy_(torch.from_numpy(self.starts[idx]))
        return torch.from_numpy(self.oplan.run_kind[idx].copy())

    def plan(self, starts, n):
        import oracle
        assert n == self.N and int(starts[-1]) == n
        mg, _ = oracle.policy(n, starts[:-1].numpy().astype(np.uint64))
        return torch.from_numpy(np.stack([mg["i"], mg["j"], mg["k"], mg["power"]], axis=1).astype(np.int64))


def _plan_worker(rank, world, port, glob, sizes, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import workloads as W
    from paper_2605_27147_b200.dist import merge_plan_dist
    off = sum(sizes[:rank])
    ops = PlanFake(glob)
    ops.sizes = sizes
    res = merge_plan_dist(W.from_numpy(glob[off:off + sizes[rank]].copy()), ops=ops)
    out_q.put((rank, res.run_start.numpy(), res.run_kind.numpy(), res.merges.numpy(), res.counts))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dtype,sizes", [
    (2, np.uint32, [4000, 3000]),
    (3, np.float32, [2500, 0, 1800]),      # an empty shard
    (3, np.uint64, [3000, 5, 2]),          # shards shorter than the halo
])
def test_merge_plan_dist_gloo(world, dtype, sizes):
    import oracle
    rng = np.random.default_rng(sum(sizes))
    N = sum(sizes)
    x = rng.integers(0, 1000, N)
    cuts = np.sort(rng.integers(0, N, 40))
    for a, b in zip(cuts[:-1], cuts[1:]):   # runs of both directions across the shard edges
        x[a:b] = np.sort(x[a:b])[::-1] if rng.random() < 0.4 else np.sort(x[a:b])
    glob = x.astype(dtype)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, glob, sizes, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=120) for _ in range(world)], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    oplan, _ = oracle.plan(glob)
    om = np.stack([oplan.merges["i"], oplan.merges["j"], oplan.merges["k"], oplan.merges["power"]], axis=1)
    for o in outs:   # the whole plan, replicated on every rank
        assert (o[1] == oplan.run_start.astype(np.int64)).all()
        assert (o[2] == oplan.run_kind).all()
        assert (o[3] == om.astype(np.int64)).all()
        assert sum(o[4]) == len(oplan.run_start)


def test_plan_host_rules():
    import oracle
    from paper_2605_27147_b200 import minrun_for
    from paper_2605_27147_b200.dist import ST_END, compose_tables, halo_from_heads, prev_owner
    for n in [1, 2, 63, 64, 65, 127, 128, 1000, 4096, 12345, 1 << 20, (1 << 30) + 7, 10 ** 12]:
        assert minrun_for(n) == oracle.minrun(n)
    # composition from START(0); END absorbs (no runs after it); empty shards pass through
    t0 = [(7 << 32) | 3, 0, 0, 0, 0, 0, 0, 0, 0]
    t2 = [0] * 7 + [(ST_END << 32) | 4, 0]
    t3 = [(1 << 32) | 9] * 9
    assert compose_tables([t0, None, t2, t3]) == ([0, 7, 7, ST_END], [3, 0, 4, 0])
    heads = [[1, 2], [3], [], [4, 5, 6]]
    sizes = [2, 1, 0, 3]
    assert [list(p) for p in halo_from_heads(0, heads, sizes, 3)] == [[3], [4, 5]]
    assert halo_from_heads(3, heads, sizes, 3) == []
    assert prev_owner(3, sizes) == 1 and prev_owner(0, sizes) == -1
