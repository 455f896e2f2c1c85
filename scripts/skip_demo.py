"""Run-skip demo: 2^28 u32 keys in 2^14 sorted segments whose value ranges are
disjoint and increasing except for one out-of-order element at each segment
start (many runs, merges mostly single-source), vs a random-runs input."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27147_b200 as vm
n = 1 << 28
dev = torch.device("cuda")
idx = torch.arange(n, device=dev, dtype=torch.int64)
seg = 1 << 14
k = idx.clone()
k[::seg] = idx[::seg] - 3  # a small descent at each segment start
k = k.clamp(min=0).to(torch.int32).view(torch.uint32)
v = idx.to(torch.int32).view(torch.uint32)
def t(keys, vals, reps=3, one=False):
    vm.test_set_mode(1 if one else 2)
    kk, vv = keys.clone(), vals.clone()
    vm.profile_enable(True)
    vm.sort_(kk, vv); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        kk.copy_(keys); vv.copy_(vals)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); vm.sort_(kk, vv); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    pr = vm.profile_read()
    vm.profile_enable(False)
    kk.copy_(keys); vv.copy_(vals)
    st = vm.sort_(kk, vv, stats=True)
    return min(ts), pr.get("merge_ms"), st["merge_cost_M"], st["runs"]
for one in (False, True):
    print(json.dumps({"input": "disjoint sorted segments", "levels_per_pass": 1 if one else 2,
                      "ms": t(k, v, one=one)}))
vm.test_set_mode(2)
