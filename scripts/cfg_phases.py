"""Phase times (ms) of one sort of each BASELINE config 1-4 (vmps profile
events) and its plan statistics.  usage: python scripts/cfg_phases.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27147_b200 as vm
import workloads as W

ws = vm.Workspace()
for c in (1, 2, 3, 4):
    k0, v0 = W.make(c, device="cuda")
    k = k0.clone(); v = None if v0 is None else v0.clone()
    st = vm.sort_(k, v, workspace=ws, stats=True)
    vm.profile_enable(True)
    for _ in range(3):
        k.copy_(k0)
        if v is not None: v.copy_(v0)
        vm.sort_(k, v, workspace=ws)
    torch.cuda.synchronize()
    pr = vm.profile_read()
    vm.profile_enable(False)
    print(json.dumps({"cfg": c, "n": k0.numel(), **{x: round(y, 3) for x, y in pr.items() if isinstance(y, float)},
                      "launches": pr.get("launches"), "runs": st["runs"], "M_over_n": st["merge_cost_M"] / k0.numel(),
                      "fused_share": st["fused_M"] / max(st["merge_cost_M"], 1), "levels": st["levels_executed"],
                      "hbm_merge_elems": st["hbm_merge_elems"]}))
    del k0, v0, k, v
