"""Scratch-bounded mode on presorted data: 2^28 u32 keys + payload in 2^14
sorted segments over disjoint increasing value ranges (one small descent at
each segment start), cap 4 sqrt(n log2 n); ms, rounds, bytes.
usage: python scripts/bd_skip_probe.py"""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27147_b200 as vm
n = 1 << 28
idx = torch.arange(n, device="cuda", dtype=torch.int64)
k0 = idx.clone()
k0[:: 1 << 14] -= 3
k0 = k0.clamp(min=0).to(torch.int32).view(torch.uint32)
v0 = idx.to(torch.int32).view(torch.uint32)
S = int(4 * math.sqrt(n * math.log2(n)))
k, v = k0.clone(), v0.clone()
st = vm.sort_(k, v, scratch=S, stats=True)
ts = []
for _ in range(3):
    k.copy_(k0); v.copy_(v0)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); vm.sort_(k, v, scratch=S); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ku, vu = k0.clone(), v0.clone()
vm.sort_(ku, vu)
print(json.dumps({"n": n, "S": S, "ms": min(ts), "rounds": st["rounds"], "M_over_n": st["merge_cost_M"] / n,
                  "equal_unbounded": bool(torch.equal(ku, k) and torch.equal(vu, v))}))
