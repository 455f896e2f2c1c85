"""Time the scratch-bounded mode against the unbounded mode (cfg2 and cfg5)."""
import json, math, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27147_b200 as vm
import workloads as W

def run(name, k0, v0, scratch, reps=3):
    k, v = k0.clone(), v0.clone()
    st = vm.sort_(k, v, scratch=scratch, stats=True)
    ts = []
    for _ in range(reps):
        k.copy_(k0); v.copy_(v0)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); vm.sort_(k, v, scratch=scratch); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    return {"case": name, "n": k0.numel(), "scratch_elems": scratch, "ms": ms,
            "Gkeys_s": k0.numel() / ms / 1e6, "scratch_bytes": st["scratch_bytes"],
            "metadata_bytes": st["metadata_bytes"], "peak_extra_device_bytes": st["peak_extra_device_bytes"],
            "block_elems": st["block_elems"], "rounds": st["rounds"]}

out = []
for cfg, lg in ((2, 24), (5, int(os.environ.get("LOG2N5", "30")))):
    n = 1 << lg
    k0, v0 = W.make(cfg, n=n, device="cuda")
    S = int(4 * math.sqrt(n * math.log2(n)))
    out.append(run(f"cfg{cfg} unbounded", k0, v0, None))
    out.append(run(f"cfg{cfg} bounded c=4", k0, v0, S))
    del k0, v0
    torch.cuda.empty_cache()
for o in out:
    print(json.dumps(o))
