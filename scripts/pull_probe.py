"""Pull-merge vs receive-buffer merge on one GPU: g sorted pieces of a cfg5
2^30 array in g separate allocations.  (a) vmps_merge_pieces straight from
the pieces; (b) what the all-to-all path does after the exchange: the pieces
copied into one receive buffer (the all-to-all's write) + vmps_merge_runs.
usage: python scripts/pull_probe.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27147_b200 as vm
import workloads as W
n = 1 << 30
dev = torch.device("cuda")
k0, v0 = W.cfg5(n=n, device=dev)
for g in (2, 4, 8):
    cuts = [n * q // g for q in range(g + 1)]
    pk = [k0[cuts[q]:cuts[q + 1]].clone() for q in range(g)]
    pv = [v0[cuts[q]:cuts[q + 1]].clone() for q in range(g)]
    for q in range(g):
        vm.sort_(pk[q], pv[q])
    counts = [cuts[q + 1] - cuts[q] for q in range(g)]
    ok = torch.empty(n, dtype=torch.uint32, device=dev); ov = torch.empty_like(ok)
    def a():
        vm.merge_pieces([t.data_ptr() for t in pk], [t.data_ptr() for t in pv], counts, ok, ov)
    rk = torch.empty(n, dtype=torch.uint32, device=dev); rv = torch.empty_like(rk)
    def b():
        for q in range(g):
            rk[cuts[q]:cuts[q + 1]].copy_(pk[q]); rv[cuts[q]:cuts[q + 1]].copy_(pv[q])
        vm.merge_runs_(rk, rv, cuts[:-1]) if hasattr(vm, "merge_runs_") else None
    def t(fn):
        fn(); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        return min(ts)
    ta = t(a)
    from paper_2605_27147_b200.dist import VmpsOps
    ops = VmpsOps()
    def b2():
        for q in range(g):
            rk[cuts[q]:cuts[q + 1]].copy_(pk[q]); rv[cuts[q]:cuts[q + 1]].copy_(pv[q])
        ops.merge_runs(rk, rv, cuts[:-1])
    tb = t(b2)
    same = bool(torch.equal(ok, rk) and torch.equal(ov, rv))
    print(json.dumps({"g": g, "pull_ms": ta, "recvbuf_copy_plus_merge_runs_ms": tb, "equal": same,
                      "pull_GBps": 16 * n / (ta / 1000) / 1e9}))
    del pk, pv
