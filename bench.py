#!/usr/bin/env python
"""Benchmark of the B200 Virtual-Memory Powersort hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one stable sort of one synthetic batch: the whole hot path (run
detection, node powers, merge tree + schedule, leaf engine, every level
merge) on cfg5 -- n = 2^30 u32 keys + u32 payload per GPU.
Timing: CUDA events on the sorting stream around each sort, W warm-up steps,
K timed steps bracketed by barrier + synchronize, max over ranks.  Between
steps the input is restored by an untimed device copy from a pristine
buffer (8 GiB, which also flushes the 126 MB L2).  Prints ONE JSON line.

--impl reference times the CPU oracle (oracle/, plain single-threaded C) on
a bounded cfg5-shaped sample per step, on the host, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sorted keys/sec (Gkeys/s) at 1/2/4/8 B200 and % of HBM merge-tree roofline"
UNIT = "Gkeys/s"
WORKLOAD = ("cfg5: n=2^30 u32 keys + u32 payload (= index) per GPU; segments 1+Geom0(1/4096), "
            "50% i.i.d. uniform unsorted / 50% sorted ascending, 5% of those reversed; "
            "unbounded scratch")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--log2n", type=int, default=30, help="per-GPU n = 2^log2n (default: cfg5's 2^30)")
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
    ap.add_argument("--native-dist", action="store_true",
                    help="N>1: the library's own NCCL protocol (vmps_sort_pairs_dist) instead of dist.py")
    ap.add_argument("--bounded-reps", type=int, default=2,
                    help="timed sorts of the scratch-bounded mode (cap 4 sqrt(n log2 n)); 0 = skip")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index: int):
        self.dev = dev_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
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
                "reasons": sorted(reasons), "samples": len(sm)}


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


def oracle_sample_rate(log2n: int, seed: int = 5):
    """Oracle (variant A, single thread) on a cfg5-shaped sample -> (Gkeys/s, seconds)."""
    import oracle
    import workloads as W
    k, v = W.cfg5(n=1 << log2n, seed=seed, device="cpu")
    kn, vn = W.to_numpy(k), W.to_numpy(v)
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
    for w in range(args.warmup):
        oracle_sample_rate(min(args.ref_sample_log2, 20), seed=100 + w)
    times = []
    for s in range(args.steps):
        _, dt = oracle_sample_rate(args.ref_sample_log2, seed=5 + s)
        times.append(dt)
    ms = 1000 * statistics.mean(times)
    n_s = 1 << args.ref_sample_log2
    val = n_s / (ms / 1000) / 1e9
    sample = (f"cfg5-shaped sample of n=2^{args.ref_sample_log2} per step (seeds 5..{4 + args.steps}); "
              "oracle variant A (copy-merge), single thread")
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
           "config": {"workload": WORKLOAD, "sample_n": n_s},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": sample, "cpu": model, "host_cores": ncpu},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2605_27147_b200 as vm
    import workloads as W
    from paper_2605_27147_b200 import build as vbuild

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
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

    n = 1 << args.log2n
    keys0, vals0 = W.cfg5(n=n, device=dev, rank=rank)
    keys = torch.empty_like(keys0)
    vals = torch.empty_like(vals0)
    ws = vm.Workspace()
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    if world > 1 and args.native_dist:
        # native protocol (csrc/comm.cu): NCCL communicator owned by libvmps
        uid = [vm.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ncomm = vm.Comm(rank, world, uid[0], local)

        def do_sort():
            vm.sort_dist_native_(ncomm, keys, vals, workspace=ws)
    elif world > 1 and args.pull_dist:
        # exchange fused with the final merge: pieces read from peer memory
        from paper_2605_27147_b200.dist import sort_dist_pull

        def do_sort():
            res = sort_dist_pull(keys, vals)
            keys.copy_(res.keys)
            vals.copy_(res.vals)
    elif world > 1:
        from paper_2605_27147_b200.dist import sort_dist_

        def do_sort():
            sort_dist_(keys, vals)
    else:
        def do_sort():
            vm.sort_(keys, vals, workspace=ws)

    # warm-up (untimed)
    keys.copy_(keys0)
    vals.copy_(vals0)
    stats = vm.sort_(keys, vals, workspace=ws, stats=True)  # local plan statistics
    for w in range(max(args.warmup, 1)):
        keys.copy_(keys0)
        vals.copy_(vals0)
        do_sort()
    torch.cuda.synchronize()

    # timed steps
    vm.profile_enable(True)
    clocks = ClockSampler(local)
    step_ms, merge_ms, merge_bytes, phases, launches = [], [], [], [], 0
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    for s in range(args.steps):
        keys.copy_(keys0)
        vals.copy_(vals0)
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
            merge_bytes.append(pr["merge_bytes"])
            phases.append(pr)
    barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    vm.profile_enable(False)

    # verify the last output (exact stable-sort properties on device)
    a = keys.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    pv = vals.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    ok = bool((a[1:] >= a[:-1]).all())
    if n * world <= (1 << 32):  # payload = global index is unique: stability is checkable
        ok = ok and bool(((pv[1:] > pv[:-1]) | (a[1:] != a[:-1])).all())
    if world > 1:  # shard boundaries: last of rank p <= first of rank p+1
        ends = torch.stack([a[0], a[-1]])
        allends = [torch.zeros_like(ends) for _ in range(world)]
        dist.all_gather(allends, ends)
        ok = ok and all(int(allends[q][1]) <= int(allends[q + 1][0]) for q in range(world - 1))
    del a, pv

    t_local = statistics.mean(step_ms)
    t = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = n * world / (ms / 1000) / 1e9

    peak, peak_src = load_peaks()
    mm = statistics.mean(merge_ms) if merge_ms else None
    mb = statistics.mean(merge_bytes) if merge_bytes else None
    w_bytes = 8
    M = stats["merge_cost_M"]
    roof = None
    if mm and mb:
        achieved = mb / (mm / 1000) / 1e9
        # DRAM bytes of the same launches from ncu (profiles/, same command at
        # the same n), per step like `achieved`; null if absent
        traffic, traffic_src = None, None
        tp = os.path.join(ROOT, "profiles", "merge_level_traffic.json")
        if os.path.exists(tp):
            try:
                tj = json.load(open(tp))
                traffic = tj.get("bytes_per_step")
                traffic_src = tj.get("source")
            except Exception:
                traffic = None
        kname = ("k_merge_level (one tree level per HBM pass; all merge launches of a step)" if args.one_level
                 else "k4_merge_level (two tree levels, up to 4-way merges, per HBM pass; all merge launches "
                      "of a step)")
        roof = {"bound": "hbm", "kernel": kname,
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_unit": "bytes per step (all level-merge launches)",
                "traffic_source": traffic_src, "peak_source": peak_src,
                "algorithmic_bytes_per_step": mb, "merge_launches_per_step": phases[-1]["merge_launches"],
                "kernel_ms_per_step": mm}
    tree = {"bytes_2wM": 2 * w_bytes * M, "M_over_n": M / n,
            "t_roof_ms_at_peak": 2 * w_bytes * M / (peak * 1e9) * 1000,
            "frac_of_roofline": (2 * w_bytes * M / (peak * 1e9) * 1000) / ms,
            "fused_M_share": stats["fused_M"] / M if M else 0.0,
            "hbm_merge_elems": stats["hbm_merge_elems"],
            "hbm_merge_bytes_over_2wM": (2 * w_bytes * stats["hbm_merge_elems"]) / (2 * w_bytes * M) if M else 0.0}
    ph = {}
    if phases:
        for key in ("plan_ms", "leaf_ms", "partition_ms", "merge_ms", "total_ms"):
            ph[key] = statistics.mean(p[key] for p in phases)

    # end-to-end through the public C-ABI host entry (vmps_sort_pairs_host):
    # every step copies its batch in from pinned host memory, sorts it and
    # copies the sorted keys + payload back out to pinned host memory.  Steps
    # rotate over NS streams with their own device buffers and workspaces, so
    # the copy engines (H2D, D2H) and the SMs work on different batches at
    # once (whole-job throughput of a stream of batches).
    e2e = None
    if not args.no_e2e and world == 1:
        NS = 3
        ks = max(NS, min(max(args.steps, 8), 12))
        hk = torch.empty(n, dtype=torch.int32, pin_memory=True).view(torch.uint32)
        hv = torch.empty(n, dtype=torch.int32, pin_memory=True).view(torch.uint32)
        hk.copy_(keys0)
        hv.copy_(vals0)
        outs = [(torch.empty(n, dtype=torch.int32, pin_memory=True).view(torch.uint32),
                 torch.empty(n, dtype=torch.int32, pin_memory=True).view(torch.uint32)) for _ in range(NS)]
        streams = [torch.cuda.Stream(dev) for _ in range(NS)]
        dbufs = [(keys, vals)] + [(torch.empty_like(keys), torch.empty_like(vals)) for _ in range(NS - 1)]
        wss = [ws] + [vm.Workspace() for _ in range(NS - 1)]

        def e2e_step(q):
            j = q % NS
            vm.sort_host_(hk, hv, device=dev, out_keys=outs[j][0], out_values=outs[j][1],
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
        # the last read-back is the exact stable sort (same input every step):
        # compare with a device-sorted reference copy
        ref_k, ref_v = keys0.clone(), vals0.clone()
        vm.sort_(ref_k, ref_v, workspace=wss[1])
        torch.cuda.synchronize()
        lo_ = outs[(ks - 1) % NS]
        ok_e2e = bool((lo_[0] == ref_k.cpu()).all()) and bool((lo_[1] == ref_v.cpu()).all())
        del ref_k, ref_v
        e2e = {"value": n / (te / 1000) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
               "ms_per_step": te, "steps": ks, "api": "vmps_sort_pairs_host (C ABI) via sort_host_",
               "pipelining": f"{NS} streams, each with its own device buffers and workspace",
               "verified": ok_e2e}
        del hk, hv, outs, dbufs, wss[1:]
    elif not args.no_e2e:
        # sharded: per rank, copy the shard in, distributed sort, copy it out
        ks = max(1, min(args.steps, 3))
        hk = torch.empty(n, dtype=torch.int32, pin_memory=True).view(torch.uint32)
        hv = torch.empty(n, dtype=torch.int32, pin_memory=True).view(torch.uint32)
        hk.copy_(keys0)
        hv.copy_(vals0)
        ok_ = torch.empty(n, dtype=torch.int32, pin_memory=True).view(torch.uint32)
        ov_ = torch.empty(n, dtype=torch.int32, pin_memory=True).view(torch.uint32)
        et = []
        for q in range(ks + 1):
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            keys.copy_(hk, non_blocking=True)
            vals.copy_(hv, non_blocking=True)
            do_sort()
            ok_.copy_(keys, non_blocking=True)
            ov_.copy_(vals, non_blocking=True)
            e1.record(stream)
            e1.synchronize()
            if q:
                et.append(e0.elapsed_time(e1))
        te = torch.tensor([statistics.mean(et)], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": n * world / (float(te.item()) / 1000) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
               "ms_per_step": float(te.item()), "steps": ks, "api": "sort_dist_ with pinned host copies"}
        del hk, hv, ok_, ov_

    bounded = None
    if world == 1 and args.bounded_reps > 0:
        import math
        S = int(4 * math.sqrt(n * math.log2(n)))
        keys.copy_(keys0)
        vals.copy_(vals0)
        bws = vm.Workspace()
        bst = vm.sort_(keys, vals, scratch=S, stats=True, workspace=bws)  # warm-up + stats
        bt = []
        for _ in range(args.bounded_reps):
            keys.copy_(keys0)
            vals.copy_(vals0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            vm.sort_(keys, vals, scratch=S, workspace=bws)
            e1.record(stream)
            e1.synchronize()
            bt.append(e0.elapsed_time(e1))
        bms = statistics.mean(bt)
        bounded = {"scratch_cap_elems": S, "c": 4, "ms_per_step": bms, "value": n / (bms / 1000) / 1e9,
                   "unit": UNIT, "slowdown_vs_unbounded": bms / ms,
                   "scratch_bytes": bst["scratch_bytes"], "metadata_bytes": bst["metadata_bytes"],
                   "peak_extra_device_bytes": bst["peak_extra_device_bytes"],
                   "unbounded_peak_extra_device_bytes": stats["peak_extra_device_bytes"],
                   "block_elems": bst["block_elems"], "rounds": bst["rounds"]}
        del bws

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        model, ncpu = cpu_info()
        v, dt = oracle_sample_rate(args.cpu_sample_log2)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"cfg5-shaped sample n=2^{args.cpu_sample_log2} (seed 5), oracle variant A, "
                         f"{dt:.1f} s single-threaded",
               "cpu": model, "host_cores": ncpu}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "u32", "data": "synthetic",
               "config": {"workload": WORKLOAD, "n_per_gpu": n, "n_total": n * world,
                          "merge_schedule": "one level per pass" if args.one_level else "two levels per pass (4-way)",
                          "key": "u32", "payload": "u32", "scratch": "unbounded",
                          "parallelism": (f"dp{world}: contiguous shards, local sort, exact splitters, "
                                          "NCCL all-to-all, local stable merge") if world > 1 else "single",
                          "timing": "CUDA events around each sort on its stream; input restored "
                                    "by an untimed 8 GiB device copy between steps (flushes L2)",
                          "runs": stats["runs"], "merge_cost_M": M, "max_power": stats["max_power"],
                          "levels_executed": stats["levels_executed"]},
               "roofline": roof, "tree_roofline": tree, "phases_ms": ph,
               "cpu_baseline": cpu, "e2e": e2e, "bounded": bounded,
               "gpu_launches": launches, "clocks": clk, "verified": ok}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
