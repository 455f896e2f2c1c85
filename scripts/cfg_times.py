"""Sort time (ms, CUDA events, median of 5 after 2 warm-ups) of BASELINE.json's
configs 1-4 at full size and of the paper's int workload (N = 10^7, S = 2 and
10^4), one JSON line.  usage: python scripts/cfg_times.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27147_b200 as vm
import workloads as W

ws = vm.Workspace()


def t(keys, vals):
    k = keys.clone(); v = None if vals is None else vals.clone()
    ts = []
    for i in range(7):
        k.copy_(keys)
        if v is not None: v.copy_(vals)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); vm.sort_(k, v, workspace=ws); e1.record(); e1.synchronize()
        if i >= 2: ts.append(e0.elapsed_time(e1))
    return round(sorted(ts)[len(ts) // 2], 3)


out = {}
for c in (1, 2, 3, 4):
    k, v = W.make(c, device="cuda")
    out[f"cfg{c}"] = t(k, v)
    del k, v
for S in (2, 10 ** 4):
    d, n = W.paper_input(S, "int", device="cuda")
    out[f"paper_S{S}"] = t(d, None)
print(json.dumps(out))
