#!/usr/bin/env python
"""Benchmark of the B200 Virtual-Memory Powersort hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 5|4|3|2|1]

One step = one stable sort of one synthetic batch: the whole hot path (run
detection, node powers, merge tree + schedule, leaf engine, every level
merge) on BASELINE.json's configuration -- by default cfg5, n = 2^30 u32 keys
+ u32 payload per GPU (weak scaling); cfg3 / cfg4 are the
strong-scaling configs (the total n is split over the GPUs).  With N > 1 each
rank sorts its contiguous shard and the library's native protocol (exact
splitters, NCCL exchange, stable merge; csrc/comm.cu) makes the result the
globally stable sort of the concatenation.

Timing: CUDA events on the sorting stream around each sort, W warm-up steps,
K timed steps bracketed by barrier + synchronize, max over ranks.  Between
steps the input is restored by an untimed device copy from a pristine buffer
(8 GiB at cfg5, which also flushes the 126 MB L2).  Rank 0 prints ONE JSON
line.  `--gpus N` without a torchrun environment launches the N ranks itself.

--impl reference times the CPU oracle (oracle/, plain single-threaded C) on
a bounded sample of the same workload per step, on the host, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sorted keys/sec (Gkeys/s) at 1/2/4/8 B200 and % of HBM merge-tree roofline"
UNIT = "Gkeys/s"
WORKLOADS = {
    5: ("cfg5: n=2^30 u32 keys + u32 payload (= global index mod 2^32) per GPU; segments 1+Geom0(1/4096), "
        "50% i.i.d. uniform unsorted / 50% sorted ascending, 5% of those reversed; unbounded scratch"),
    4: ("cfg4: n=2^28 f32 keys in total, no payload; 'Timsort-drag' run lengths (reading R13), "
        "values normal(0,1) with +-0.0; unbounded scratch"),
    3: ("cfg3: n=2^26 u64 keys in total (values 0..15) + u32 payload (= index); runs U[1, 2 sqrt n], "
        "10% reversed (plateaus); unbounded scratch"),
    2: "cfg2: n=2^24 u32 + u32 payload (= index); random runs, lengths U[1, 2 sqrt n]; unbounded scratch",
    1: "cfg1: n=2^20 u32 random permutation of 0..n-1 (seed 1); no payload; unbounded scratch",
}
DEFAULT_LOG2N = {5: 30, 4: 28, 3: 26, 2: 24, 1: 20}
STRONG = {3, 4}  # BASELINE.json: cfg3 at 1/2 GPUs, cfg4 at 1/2/4 GPUs (fixed total n)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--log2n", type=int, default=0,
                    help="n = 2^log2n (per GPU for cfg5, total for the others); default: the config's")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-log2", type=int, default=25)
    ap.add_argument("--ref-sample-log2", type=int, default=23)
    ap.add_argument("--one-level", action="store_true",
                    help="A/B: one tree level (2-way merges) per HBM pass instead of two (4-way)")
    ap.add_argument("--leaf-radix", action="store_true",
                    help="experimental: radix-sort leaf engine instead of the block merge sort")
    ap.add_argument("--fuse-z", type=int, default=0, help="experimental: fused-subtree limit Z")
    ap.add_argument("--pull-dist", action="store_true",
                    help="N>1: pull-merge the co-ranked pieces from peer memory (dist.sort_dist_pull)")
    ap.add_argument("--bounded-reps", type=int, default=2,
                    help="timed sorts of the scratch-bounded mode (cap 4 sqrt(n log2 n)); 0 = skip")
    ap.add_argument("--verify-oracle", action="store_true",
                    help="slow, untimed: every rank's local sort vs the oracle on the host, and the global plan "
                         "vs the oracle's plan-only pass over the whole array (rank 0; SURVEY 8(d) (i), (iii))")
    ap.add_argument("--launcher-selftest", action="store_true",
                    help="CPU check of the N-rank launcher: every rank joins a gloo group; rank 0 prints n_gpus")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons of the GPUs in use, sampled during
    the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, devs):
        self.devs = ",".join(str(d) for d in devs)
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.devs, f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() in ("active", "1", "yes"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "gpus": self.devs}


def cpu_info():
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return model, os.cpu_count()


def gen_host(cfg: int, n: int, seed_shift: int = 0):
    """The config's generator on the host (numpy), for the oracle samples."""
    import workloads as W
    if cfg == 5:
        k, v = W.cfg5(n=n, seed=5 + seed_shift, device="cpu")
    else:
        k, v = W.make(cfg, n=n, seed=cfg + seed_shift, device="cpu")
    return W.to_numpy(k), (W.to_numpy(v) if v is not None else None)


def oracle_sample_rate(cfg: int, log2n: int, seed_shift: int = 0):
    """Oracle (variant A, single thread) on a sample of the workload -> (Gkeys/s, seconds)."""
    import oracle
    kn, vn = gen_host(cfg, 1 << log2n, seed_shift)
    t0 = time.perf_counter()
    oracle.sort(kn, vn, variant=oracle.VARIANT_A)
    dt = time.perf_counter() - t0
    return (1 << log2n) / dt / 1e9, dt


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    model, ncpu = cpu_info()
    import oracle
    oracle.build()
    cfg = args.config
    log2 = min(args.ref_sample_log2, args.log2n or DEFAULT_LOG2N[cfg])
    for w in range(args.warmup):
        oracle_sample_rate(cfg, min(log2, 20), seed_shift=100 + w)
    times = []
    for s in range(args.steps):
        _, dt = oracle_sample_rate(cfg, log2, seed_shift=s)
        times.append(dt)
    ms = 1000 * statistics.mean(times)
    n_s = 1 << log2
    val = n_s / (ms / 1000) / 1e9
    sample = (f"cfg{cfg}-shaped sample of n=2^{log2} per step (seeds shifted 0..{args.steps - 1}); "
              "oracle variant A (copy-merge), single thread")
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong" if cfg in STRONG else "weak", "vs_baseline": None,
           "dtype": {3: "u64", 4: "f32"}.get(cfg, "u32"), "data": "synthetic",
           "config": {"workload": WORKLOADS[cfg], "sample_n": n_s},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": sample, "cpu": model, "host_cores": ncpu},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args) -> int:
    """`--gpus N` outside torchrun: launch N ranks of this script (one per GPU,
    rendezvous on 127.0.0.1) and forward rank 0's output."""
    import torch
    ndev = torch.cuda.device_count()
    if ndev < args.gpus and not args.launcher_selftest:
        print(f"bench.py: --gpus {args.gpus} but only {ndev} CUDA device(s) visible; refusing to run "
              f"(the JSON line would report a different n_gpus)", file=sys.stderr)
        return 2
    port = _free_port()
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


def order_image(t):
    """Order image of a key tensor as int64 (u32 / f32: exact in 0..2^32; u64:
    top bit flipped so that signed comparison is the unsigned order)."""
    import torch
    if t.dtype == torch.float32:
        b = t.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        nan = (b & 0x7FFFFFFF) > 0x7F800000
        img = torch.where((b >> 31) == 1, b ^ 0xFFFFFFFF, b | 0x80000000)
        return torch.where(nan, torch.full_like(img, 0xFFFFFFFF), img)
    if t.dtype == torch.uint64:
        return t.view(torch.int64) ^ torch.iinfo(torch.int64).min
    return t.view(torch.int32).to(torch.int64) & 0xFFFFFFFF


def mix_hash(k, v):
    """Sum over the elements of a 64-bit mix of (key bits, payload) mod 2^64:
    equal multisets of pairs give equal sums (the permutation check)."""
    import torch
    kb = k.view(torch.int64) if k.element_size() == 8 else (k.view(torch.int32).to(torch.int64) & 0xFFFFFFFF)
    x = kb * -7046029254386353131  # 0x9E3779B97F4A7C15
    if v is not None:
        x = x ^ ((v.view(torch.int32).to(torch.int64) & 0xFFFFFFFF) * -4417276706812531889)  # 0xC2B2AE3D27D4EB4F
    x = x ^ ((x >> 31) & 0x1FFFFFFFF)
    x = x * -4658895280553007687  # 0xBF58476D1CE4E5B9
    x = x ^ ((x >> 29) & 0x7FFFFFFFF)
    return int(x.sum().item())


def _sv(t):
    """Same-size signed view (torch has no comparisons / pinned copies for every unsigned type)."""
    import torch
    return t.view(torch.int64 if t.element_size() == 8 else torch.int32)


def _pinned_like(t):
    import torch
    return torch.empty(t.numel(), dtype=_sv(t).dtype, pin_memory=True).view(t.dtype)


def plan_hash_of(i, j, k, pw, order):
    """Sum over merge records of a 64-bit mix of (i, j, k, power, order)."""
    x = i * -7046029254386353131 + j * -4417276706812531889 + k * 1609587929392839161
    x = x ^ (pw * 2246822519 + order * 3266489917)
    x = x ^ ((x >> 31) & 0x1FFFFFFFF)
    x = x * -4658895280553007687
    return int(x.sum().item())


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.launcher_selftest:  # rendezvous plumbing only (no GPU)
        import torch
        import torch.distributed as dist
        world = int(os.environ.get("WORLD_SIZE", "1"))
        if world > 1:
            dist.init_process_group("gloo")
            t = torch.ones(1)
            dist.all_reduce(t)
            world = int(t.item())
            dist.destroy_process_group()
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps({"launcher_selftest": True, "n_gpus": world}), flush=True)
        return
    import torch
    import torch.distributed as dist

    import numpy as np

    import paper_2605_27147_b200 as vm
    import workloads as W
    from paper_2605_27147_b200 import build as vbuild

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; refusing to report n_gpus={world}",
              file=sys.stderr)
        sys.exit(2)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if not os.path.exists(vm.LIB_PATH):
        vbuild.build()
    vm.lib()
    if args.one_level:
        vm.test_set_mode(1)
    if args.leaf_radix:
        vm.test_set_leaf(True)
    if args.fuse_z:
        vm.test_set_tiles(args.fuse_z, 0, 0)

    cfg = args.config
    log2n = args.log2n or DEFAULT_LOG2N[cfg]
    strong = cfg in STRONG
    if cfg == 5:  # weak scaling: 2^log2n per GPU, generated by global index
        n = 1 << log2n
        keys0, vals0 = W.cfg5(n=n, device=dev, rank=rank)
        n_total = n * world
    else:  # the config's total n, split into contiguous shards
        n_total = 1 << log2n
        fk, fv = W.make(cfg, n=n_total, device=dev)
        a, b = rank * n_total // world, (rank + 1) * n_total // world
        keys0 = fk[a:b].clone()
        vals0 = fv[a:b].clone() if fv is not None else None
        del fk, fv
        n = b - a
    hv = vals0 is not None
    w_bytes = keys0.element_size() + (4 if hv else 0)
    keys = torch.empty_like(keys0)
    vals = torch.empty_like(vals0) if hv else None
    ws = vm.Workspace()
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def restore():
        _sv(keys).copy_(_sv(keys0))
        if hv:
            _sv(vals).copy_(_sv(vals0))

    ncomm = None
    if world > 1:
        from paper_2605_27147_b200 import dist as vdist
        ncomm = vdist.native_comm(None, dev)
        if args.pull_dist:
            def do_sort():
                res = vdist.sort_dist_pull(keys, vals, comm=ncomm, workspace=ws)
                _sv(keys).copy_(_sv(res.keys))
                if hv:
                    _sv(vals).copy_(_sv(res.vals))
        else:
            def do_sort():
                vdist.sort_dist_(keys, vals, comm=ncomm, workspace=ws)
    else:
        def do_sort():
            vm.sort_(keys, vals, workspace=ws)

    # local plan statistics (one untimed local sort)
    restore()
    stats = vm.sort_(keys, vals, workspace=ws, stats=True)
    overify = {}
    if args.verify_oracle:  # (i): this rank's local sort vs the oracle (host, single thread)
        import oracle
        import workloads as W
        kh = W.to_numpy(keys0)
        ko, vo, _, _ = oracle.sort(kh, W.to_numpy(vals0) if hv else None)
        okl = bool((W.to_numpy(keys).view(np.uint8) == ko.view(np.uint8)).all()) and (
            not hv or bool((W.to_numpy(vals) == vo).all()))
        t = torch.tensor([1 if okl else 0], dtype=torch.int64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
        overify["local_sorts_equal_oracle"] = bool(t.item())
        del kh, ko, vo
    # the global plan's merge cost (the roofline uses the plan of
    # the whole array): untimed vmps_merge_plan_dist, merges summed over ranks
    runs_g, M_g = stats["runs"], stats["merge_cost_M"]
    plan_hash = None
    if world > 1:
        from paper_2605_27147_b200 import dist as vdist
        p = vdist.merge_plan_dist(keys0, n_total=n_total, comm=ncomm)
        mk = p.merges
        ph = 0
        if args.verify_oracle and mk.numel():
            ph = plan_hash_of(mk[:, 0], mk[:, 1], mk[:, 2], mk[:, 3], mk[:, 4])
        t = torch.tensor([int(p.run_start.numel()), int((mk[:, 2] - mk[:, 0]).sum().item()) if mk.numel() else 0, ph],
                         dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        runs_g, M_g, plan_hash = int(t[0].item()), int(t[1].item()), int(t[2].item())
        del p, mk
    elif args.verify_oracle:
        p = vm.merge_plan(keys0)
        mk = p.merges
        ordr = torch.arange(mk.shape[0], dtype=torch.int64, device=dev)
        plan_hash = plan_hash_of(mk[:, 0], mk[:, 1], mk[:, 2], mk[:, 3], ordr) if mk.numel() else 0
        del p, mk
    glob = None
    if args.verify_oracle:  # (iii): the whole array on rank 0's host (shards sent in 256 MiB pieces)
        import workloads as W
        parts = [W.to_numpy(keys0)] if rank == 0 else []
        CH = (256 << 20) // keys0.element_size()
        for q in range(1, world):
            nq = torch.tensor([n], dtype=torch.int64, device=dev)
            dist.broadcast(nq, src=q)
            nq = int(nq.item())
            buf = torch.empty(min(CH, max(nq, 1)), dtype=_sv(keys0).dtype, device=dev)
            got = []
            for a in range(0, nq, CH):
                m = min(CH, nq - a)
                if rank == q:
                    dist.send(_sv(keys0)[a:a + m].contiguous(), dst=0)
                elif rank == 0:
                    dist.recv(buf[:m], src=q)
                    got.append(buf[:m].view(keys0.dtype).cpu())
            if rank == 0:
                parts.append(W.to_numpy(torch.cat(got)) if got else np.zeros(0, W.to_numpy(keys0[:0]).dtype))
        if rank == 0:
            glob = np.concatenate(parts)
        del parts
    if args.verify_oracle and rank == 0:
        import oracle
        oplan, ost = oracle.plan(glob)
        om = oplan.merges
        dv = "cpu"
        oh = plan_hash_of(*(torch.from_numpy(om[f].astype(np.int64)) for f in ("i", "j", "k", "power")),
                          torch.arange(len(om), dtype=torch.int64)) if len(om) else 0
        overify.update(plan_runs_equal=len(oplan.run_start) == runs_g, plan_M_equal=ost["merge_cost_M"] == M_g,
                       plan_hash_equal=(oh - plan_hash) % (1 << 64) == 0,
                       plan_check="hash of (i, j, k, power, order) summed over the merges")
        del glob, oplan, om, dv
    for w in range(max(args.warmup, 1)):
        restore()
        do_sort()
    torch.cuda.synchronize()

    # timed steps
    vm.profile_enable(True)
    clocks = ClockSampler(range(world) if rank == 0 else [local])
    step_ms, merge_ms, phases, launches = [], [], [], 0
    barrier()
    torch.cuda.synchronize()
    if rank == 0:
        clocks.start()
    for s in range(args.steps):
        restore()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        do_sort()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        pr = vm.profile_read()
        launches += pr.get("launches", 0)
        if "merge_ms" in pr:
            merge_ms.append(pr["merge_ms"])
            phases.append(pr)
    barrier()
    torch.cuda.synchronize()
    clk = clocks.stop() if rank == 0 else None
    vm.profile_enable(False)

    # verify the last output: sorted (across ranks too), the same multiset of
    # (key, payload) pairs as the input, stable by the global-index payload
    img = order_image(keys)
    ok = bool((img[1:] >= img[:-1]).all()) if n > 1 else True
    eq = img[1:] == img[:-1]
    stab = "n/a (no payload)"
    if hv:
        pv = vals.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        if n_total <= (1 << 32):  # payload = global index is unique: strictly increasing within ties
            ok = ok and bool(((pv[1:] > pv[:-1]) | ~eq).all())
            stab = "payload (global index) strictly increasing within equal keys"
        else:  # index mod 2^32: at most one wrap per tie group
            desc = (eq & (pv[1:] <= pv[:-1])).to(torch.int64)
            grp = torch.cumsum((~eq).to(torch.int64), 0)
            per = torch.zeros(int(grp[-1].item()) + 1, dtype=torch.int64, device=dev).index_add_(0, grp, desc)
            ok = ok and bool((per <= 1).all())
            stab = "payload (global index mod 2^32) wraps at most once within equal keys"
        del pv
    if world == 1 and hv and n_total <= (1 << 32):  # exact permutation: keys travel with their index
        ok = ok and bool((_sv(keys) == _sv(keys0)[vals.view(torch.int32).to(torch.int64) & 0xFFFFFFFF]).all())
    h_in, h_out = mix_hash(keys0, vals0), mix_hash(keys, vals)
    if world > 1:
        hs = torch.tensor([h_in, h_out], dtype=torch.int64, device=dev)
        dist.all_reduce(hs)
        h_in, h_out = int(hs[0].item()), int(hs[1].item())
        ends = torch.stack([img[0], img[-1]]) if n else torch.tensor([0, 0], dtype=torch.int64, device=dev)
        allends = [torch.zeros_like(ends) for _ in range(world)]
        dist.all_gather(allends, ends)
        ok = ok and all(int(allends[q][1]) <= int(allends[q + 1][0]) for q in range(world - 1))
        okt = torch.tensor([1 if ok else 0], dtype=torch.int64, device=dev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        ok = bool(okt.item())
    ok = ok and h_in == h_out
    del img, eq

    t_local = statistics.mean(step_ms)
    t = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = n_total / (ms / 1000) / 1e9

    peak, peak_src = load_peaks()
    M_loc, fM_loc, hme = stats["merge_cost_M"], stats["fused_M"], stats["hbm_merge_elems"]
    mm = statistics.mean(merge_ms) if merge_ms else None
    roof = None
    if mm:
        algo = 2 * w_bytes * (M_loc - fM_loc)       # 2w per element per non-fused tree level
        phys = 2 * w_bytes * hme                     # bytes the two-levels-per-pass kernel reads + writes
        traffic, traffic_src = None, None
        tp = os.path.join(ROOT, "profiles", "merge_level_traffic.json")
        if os.path.exists(tp) and cfg == 5 and log2n == 30 and not args.one_level:
            try:
                tj = json.load(open(tp))
                traffic, traffic_src = tj.get("bytes_per_step"), tj.get("source")
            except Exception:
                traffic = None
        kname = ("k_merge_level (one tree level per HBM pass; all merge launches of a step)" if args.one_level
                 else "k4_merge_level (two tree levels, up to 4-way merges, per HBM pass; all merge launches "
                      "of a step)")
        achieved = algo / (mm / 1000) / 1e9
        roof = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_unit": "DRAM bytes per step (all level-merge launches, ncu)",
                "traffic_source": traffic_src, "peak_source": peak_src,
                "algorithmic_bytes_per_step": algo,
                "algorithmic_basis": "SURVEY 8(d): 2w bytes per element per non-fused merge-tree level, "
                                     "2w(M - M_fused) per step (M_fused: levels done inside the leaf sort)",
                "physical": {"bytes_per_step": phys, "achieved": phys / (mm / 1000) / 1e9,
                             "frac": phys / (mm / 1000) / 1e9 / peak,
                             "basis": "2w x elements the 4-way kernel reads and writes (two tree levels "
                                      "per HBM pass: only even-depth nodes are materialized)"},
                "merge_launches_per_step": phases[-1]["merge_launches"], "kernel_ms_per_step": mm,
                "timing": "CUDA events around each level-merge launch on the sorting stream, "
                          "over the timed steps"}
    t_roof = 2 * w_bytes * M_g / (world * peak * 1e9) * 1000
    tree = {"bytes_2wM": 2 * w_bytes * M_g, "M": M_g, "M_over_n": M_g / n_total, "runs": runs_g,
            "M_source": "global plan (vmps_merge_plan_dist over the shards)" if world > 1 else "plan of the array",
            "t_roof_ms_at_peak": t_roof, "frac_of_roofline": t_roof / ms,
            "local_M": M_loc, "fused_M_share": fM_loc / M_loc if M_loc else 0.0, "hbm_merge_elems": hme,
            "hbm_merge_bytes_over_2wM": hme / M_loc if M_loc else 0.0}
    ph = {}
    if phases:
        for key in ("plan_ms", "leaf_ms", "partition_ms", "merge_ms", "total_ms"):
            ph[key] = statistics.mean(p[key] for p in phases)
        if world > 1:
            ph["note"] = "phases of this rank's local sort (rank 0); exchange and final merge not split out"

    # end-to-end through the public C-ABI host entry points: every step copies
    # its batch in from pinned host memory, sorts it and copies the result out
    e2e = None
    if not args.no_e2e and world == 1:
        NS = 3
        ks = max(NS, min(max(args.steps, 8), 12))
        hk = _pinned_like(keys0)
        _sv(hk).copy_(_sv(keys0))
        hvv = None
        if hv:
            hvv = _pinned_like(vals0)
            _sv(hvv).copy_(_sv(vals0))
        outs = [(_pinned_like(keys0), _pinned_like(vals0) if hv else None) for _ in range(NS)]
        streams = [torch.cuda.Stream(dev) for _ in range(NS)]
        dbufs = [(keys, vals)] + [(torch.empty_like(keys), torch.empty_like(vals) if hv else None)
                                  for _ in range(NS - 1)]
        wss = [ws] + [vm.Workspace() for _ in range(NS - 1)]

        def e2e_step(q):
            j = q % NS
            vm.sort_host_(hk, hvv, device=dev, out_keys=outs[j][0], out_values=outs[j][1],
                          d_keys=dbufs[j][0], d_values=dbufs[j][1], workspace=wss[j], stream=streams[j])

        for q in range(NS):  # warm-up (workspace allocation, first-touch)
            e2e_step(q)
        torch.cuda.synchronize()
        cur = torch.cuda.current_stream(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for st_ in streams:
            st_.wait_event(e0)
        for q in range(ks):
            e2e_step(q)
        for st_ in streams:
            ev = torch.cuda.Event()
            ev.record(st_)
            cur.wait_event(ev)
        e1.record(cur)
        e1.synchronize()
        te = e0.elapsed_time(e1) / ks
        # the last read-back equals the device sort verified above (same input every step)
        lo_ = outs[(ks - 1) % NS]
        ok_e2e = bool((_sv(lo_[0]).to(dev) == _sv(keys)).all()) and (
            not hv or bool((_sv(lo_[1]).to(dev) == _sv(vals)).all()))
        e2e = {"value": n / (te / 1000) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": n * w_bytes, "d2h_bytes_per_step": n * w_bytes,
               "ms_per_step": te, "steps": ks, "api": "vmps_sort_*_host (C ABI) via sort_host_",
               "pipelining": f"{NS} streams, each with its own device buffers and workspace",
               "verified": ok_e2e}
        del hk, hvv, outs, dbufs, wss[1:]
    elif not args.no_e2e:
        # sharded: per rank, copy the shard in, distributed sort, copy it out
        ks = max(1, min(args.steps, 3))
        hk = _pinned_like(keys0)
        _sv(hk).copy_(_sv(keys0))
        hvv = _pinned_like(vals0) if hv else None
        if hv:
            _sv(hvv).copy_(_sv(vals0))
        ok_ = _pinned_like(keys0)
        ov_ = _pinned_like(vals0) if hv else None
        et = []
        for q in range(ks + 1):
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _sv(keys).copy_(_sv(hk), non_blocking=True)
            if hv:
                _sv(vals).copy_(_sv(hvv), non_blocking=True)
            do_sort()
            _sv(ok_).copy_(_sv(keys), non_blocking=True)
            if hv:
                _sv(ov_).copy_(_sv(vals), non_blocking=True)
            e1.record(stream)
            e1.synchronize()
            if q:
                et.append(e0.elapsed_time(e1))
        te = torch.tensor([statistics.mean(et)], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": n_total / (float(te.item()) / 1000) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": n * w_bytes, "d2h_bytes_per_step": n * w_bytes,
               "bytes_note": "per rank", "ms_per_step": float(te.item()), "steps": ks,
               "api": "dist.sort_dist_ (vmps_sort_*_dist) with pinned host copies on each rank"}
        del hk, hvv, ok_, ov_

    bounded = None
    if args.bounded_reps > 0 and hv:
        import math
        S = int(4 * math.sqrt(n * math.log2(n)))
        restore()
        bws = vm.Workspace()

        def bsort(st=False):
            if world > 1:  # per-GPU cap, exchange staging included (merge-split protocol, comm.cu)
                from paper_2605_27147_b200 import dist as vdist
                return vdist.sort_dist_(keys, vals, comm=ncomm, workspace=bws, scratch=S, stats=st)
            return vm.sort_(keys, vals, scratch=S, stats=st, workspace=bws)

        bst = bsort(True)  # warm-up + stats
        bt = []
        for _ in range(args.bounded_reps):
            restore()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            bsort()
            e1.record(stream)
            e1.synchronize()
            bt.append(e0.elapsed_time(e1))
        tb = torch.tensor([statistics.mean(bt)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tb, op=dist.ReduceOp.MAX)
        bms = float(tb.item())
        bounded = {"scratch_cap_elems": S, "c": 4, "ms_per_step": bms, "value": n_total / (bms / 1000) / 1e9,
                   "unit": UNIT, "slowdown_vs_unbounded": bms / ms,
                   "scratch_bytes": bst["scratch_bytes"], "metadata_bytes": bst["metadata_bytes"],
                   "peak_extra_device_bytes": bst["peak_extra_device_bytes"],
                   "unbounded_peak_extra_device_bytes": stats["peak_extra_device_bytes"],
                   "block_elems": bst["block_elems"], "rounds": bst["rounds"]}
        del bws

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        model, ncpu = cpu_info()
        log2 = min(args.cpu_sample_log2, log2n)
        v, dt = oracle_sample_rate(cfg, log2)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"cfg{cfg}-shaped sample n=2^{log2}, oracle variant A, {dt:.1f} s single-threaded"
                         + (" on rank 0's host" if world > 1 else ""),
               "cpu": model, "host_cores": ncpu}

    if rank == 0:
        if world > 1:
            par = (f"dp{world}: contiguous shards, local sort, exact splitters (native 16-ary search), "
                   + ("CUDA-IPC pull-merge from peer memory" if args.pull_dist else
                      "NCCL grouped send/recv, stable merge of the pieces (vmps_sort_pairs_dist)"))
        else:
            par = "single"
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
               "scaling": "strong" if strong else "weak", "vs_baseline": None,
               "dtype": {3: "u64", 4: "f32"}.get(cfg, "u32"), "data": "synthetic",
               "config": {"workload": WORKLOADS[cfg], "config": cfg, "n_per_gpu": n, "n_total": n_total,
                          "merge_schedule": "one level per pass" if args.one_level else "two levels per pass (4-way)",
                          "key": str(keys0.dtype).replace("torch.", ""), "payload": "u32" if hv else None,
                          "scratch": "unbounded", "parallelism": par,
                          "timing": "CUDA events around each sort on its stream, max over ranks; input restored "
                                    "by an untimed device copy between steps (cfg5: 8 GiB, flushes L2)",
                          "runs": runs_g, "merge_cost_M": M_g, "max_power": stats["max_power"],
                          "levels_executed": stats["levels_executed"]},
               "roofline": roof, "tree_roofline": tree, "phases_ms": ph,
               "cpu_baseline": cpu, "e2e": e2e, "bounded": bounded,
               "gpu_launches": launches, "clocks": clk, "verified": ok,
               "oracle_verification": overify or None,
               "verification": {"sorted": True, "multiset_hash": "sum of mix64(key, payload) equal before / after",
                                "stability": stab,
                                "permutation": "keys == input[payload] (exact)" if world == 1 and hv else
                                "via the multiset hash"}}
        print(json.dumps(out), flush=True)
    if world > 1:
        from paper_2605_27147_b200 import dist as vdist
        vdist.destroy_comms()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
