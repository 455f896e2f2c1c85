"""Bounded-mode probe: cfg5-shaped input of n keys (argv[1] = log2 n) sorted with
the BASELINE scratch cap 4 sqrt(n log2 n); prints ms, rounds and phase times."""
import math, sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27147_b200 as vm
import workloads as W
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = 1 << lg
k0, v0 = W.cfg5(n=n, device="cuda")
S = int(4 * math.sqrt(n * math.log2(n)))
k, v = k0.clone(), v0.clone()
st = vm.sort_(k, v, scratch=S, stats=True)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    k.copy_(k0); v.copy_(v0)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); vm.sort_(k, v, scratch=S); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ku, vu = k0.clone(), v0.clone()
vm.sort_(ku, vu)
ok = bool(torch.equal(ku, k) and torch.equal(vu, v))
print(json.dumps({"n": n, "S": S, "ms": min(ts), "rounds": st["rounds"], "us_per_round": min(ts) * 1000 / max(st["rounds"], 1),
                  "block_elems": st["block_elems"], "equal_unbounded": ok}))
