"""Multi-GPU protocol, CPU side.  The native protocol lives in
libvmps (csrc/comm.cu); its host arithmetic -- the 16-ary splitter search
over the key order image, the tie split in rank order and the composition of
the shards' run-detection transfer tables -- is exported through the C ABI
(vmps_splitter_probes / vmps_splitter_update / vmps_split_points /
vmps_compose_tables) and needs no GPU.  Here 2 and 3 gloo ranks on CPU run the
protocol's collective skeleton around those C functions, with NumPy stand-ins
(test-side only) for the device steps (local sort, rank counts, merge of the
received pieces), and the result is checked against the stable sort of the
concatenated shards.  The device path with several ranks runs in
tests/test_gpu_comm.py (virtual ranks on one GPU)."""
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


def img_max(dtype) -> int:
    return (1 << 64) - 1 if dtype == np.uint64 else (1 << 32) - 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _protocol(rank, world, k, v):
    """One rank of the sharded sort: NumPy stand-ins for the device steps,
    gloo for the collectives, libvmps's host arithmetic for the decisions."""
    import paper_2605_27147_b200 as vm
    idx = np.argsort(image_np(k), kind="stable")          # local sort (stand-in)
    k, v = k[idx], v[idx]
    img = image_np(k)
    sizes = [None] * world
    dist.all_gather_object(sizes, len(k))
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    m = world - 1
    Rt = [int(off[t + 1]) for t in range(m)]
    lo, hi = [0] * m, [img_max(k.dtype)] * m
    rounds = 0
    while True:
        probes, base = vm.splitter_probes(lo, hi)
        if not probes:
            break
        rounds += 1
        le = torch.from_numpy(np.searchsorted(img, np.array(probes, np.uint64), side="right").astype(np.int64))
        dist.all_reduce(le)                                 # counts summed over the ranks
        lo, hi = vm.splitter_update(lo, hi, Rt, probes, base, le.tolist())
    vstar = np.array(lo, np.uint64)
    cnt = (np.searchsorted(img, vstar, side="left").tolist(), np.searchsorted(img, vstar, side="right").tolist())
    allc = [None] * world
    dist.all_gather_object(allc, cnt)
    cut = [[0] * (world + 1) for _ in range(world)]
    for q in range(world):
        cut[q][world] = sizes[q]
    for t in range(m):
        pts = vm.split_points(Rt[t], [allc[q][0][t] for q in range(world)], [allc[q][1][t] for q in range(world)])
        for q in range(world):
            cut[q][t + 1] = pts[q]
    pieces = [(k[cut[rank][p]:cut[rank][p + 1]], v[cut[rank][p]:cut[rank][p + 1]]) for p in range(world)]
    got = [None] * world
    dist.all_gather_object(got, pieces)                     # exchange (stand-in for send / recv)
    rk = np.concatenate([got[q][rank][0] for q in range(world)])
    rv = np.concatenate([got[q][rank][1] for q in range(world)])
    j = np.argsort(image_np(rk), kind="stable")             # merge in source-rank order (stand-in)
    return rk[j], rv[j], rounds, cut


def _worker(rank, world, port, shards, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    k, v = shards[rank]
    rk, rv, rounds, cut = _protocol(rank, world, k, v)
    out_q.put((rank, rk, rv, rounds, cut))
    dist.destroy_process_group()


def _run(world, shards):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shards, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(outs, key=lambda x: x[0])


@pytest.mark.parametrize("world,dtype,sizes", [
    (2, np.uint32, [3000, 3000]),
    (2, np.uint64, [2500, 2500]),
    (2, np.float32, [2000, 2000]),
    (3, np.uint32, [1000, 2500, 1700]),   # unequal shards
    (3, np.uint32, [1500, 0, 900]),       # an empty shard
])
def test_sort_dist_gloo(world, dtype, sizes):
    rng = np.random.default_rng(world * 100 + len(sizes) + sum(sizes))
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
    # rank p keeps its element count: global output ranks [off_p, off_p + n_p)
    for p, o in enumerate(outs):
        assert len(o[1]) == sizes[p]
        assert o[3] <= 8 if dtype != np.uint64 else o[3] <= 16   # 16-ary search: 32 / 64 bits


def test_split_points_rule():
    import paper_2605_27147_b200 as vm
    # ranks 0..2 with lt/le counts at v*: the tie group is taken in rank order
    assert vm.split_points(10, [3, 2, 1], [6, 6, 4]) == [6, 3, 1]   # need 4 ties: 3 from r0, 1 from r1
    assert vm.split_points(6, [3, 2, 1], [6, 6, 4]) == [3, 2, 1]    # no ties taken
    assert vm.split_points(16, [3, 2, 1], [6, 6, 4]) == [6, 6, 4]   # all ties taken


def test_splitter_search_brute_force():
    """The 16-ary search ends at v* = the least image v with #{<= v} >= R, for
    every R, on small multisets (brute force over the value range)."""
    import paper_2605_27147_b200 as vm
    rng = np.random.default_rng(9)
    for trial in range(60):
        img = np.sort(rng.integers(0, 40, int(rng.integers(1, 60)))).astype(np.uint64)
        Rs = sorted(set(int(x) for x in rng.integers(1, len(img) + 1, 3)))
        lo, hi = [0] * len(Rs), [(1 << 32) - 1] * len(Rs)
        while True:
            pr, base = vm.splitter_probes(lo, hi)
            if not pr:
                break
            le = np.searchsorted(img, np.array(pr, np.uint64), side="right").tolist()
            lo, hi = vm.splitter_update(lo, hi, Rs, pr, base, le)
        for t, Rv in enumerate(Rs):
            want = min(v for v in range(41) if int((img <= v).sum()) >= Rv)
            assert lo[t] == hi[t] == want


def test_compose_tables_rule():
    """Composition from START(0); END (255) absorbs (no runs after it); empty
    shards pass through (vmps_compose_tables)."""
    import paper_2605_27147_b200 as vm
    ns = 9
    t0 = [(7 << 32) | 3, 0, 0, 0, 0, 0, 0, 0, 0]
    t2 = [0] * 7 + [(255 << 32) | 4, 0]
    t3 = [(1 << 32) | 9] * 9
    entry, count = vm.compose_tables([t0, None, t2, t3], [10, 0, 5, 7], ns)
    assert entry == [0, 7, 7, 255] and count == [3, 0, 4, 0]


def test_bench_launcher_world2():
    """`bench.py --gpus N` outside torchrun launches N ranks itself (127.0.0.1
    rendezvous); the gloo self-test of that plumbing reports n_gpus = N."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--launcher-selftest"],
                         capture_output=True, text=True, timeout=180, env=env)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2
