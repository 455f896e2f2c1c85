"""Scratch-bounded cfg5 (n = 2^LOG2N, cap 4 sqrt(n log2 n)): time, rounds and
metadata of the dyadic-cell mode for a sweep of cell sizes (test hook
vmps_test_set_bd_chunk), and the one-piece bounded mode, all checked against
the unbounded sort."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27147_b200 as vm
import workloads as W
lg = int(os.environ.get("LOG2N", "30"))
n = 1 << lg
k0, v0 = W.cfg5(n=n, device="cuda")
S = int(4 * math.sqrt(n * math.log2(n)))
ku, vu = k0.clone(), v0.clone()
stu = vm.sort_(ku, vu, stats=True)
L = vm.lib()
for ch in [int(x) for x in os.environ.get("CHUNKS", "20,21,22,23,24,31").split(",")]:
    L.vmps_test_set_bd_chunk(min(1 << ch, 0xFFFFFFFF))
    k, v = k0.clone(), v0.clone()
    st = vm.sort_(k, v, scratch=S, stats=True)
    torch.cuda.synchronize()
    ok = bool(torch.equal(ku, k) and torch.equal(vu, v))
    ts = []
    for _ in range(2):
        k.copy_(k0); v.copy_(v0)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); vm.sort_(k, v, scratch=S); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"log2_cell": ch, "ms": min(ts), "rounds": st["rounds"], "M": st["merge_cost_M"],
                      "M_unbounded": stu["merge_cost_M"], "metadata_MB": st["metadata_bytes"] / 1e6,
                      "equal_unbounded": ok}), flush=True)
    del k, v
    torch.cuda.empty_cache()
L.vmps_test_set_bd_chunk(0)
