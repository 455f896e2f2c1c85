"""One sort of the paper's int workload (N = 10^7, S = argv[1]) after a warm-up,
for launch-list profiling of the small-n regime."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27147_b200 as vm
import workloads as W
S = int(sys.argv[1]) if len(sys.argv) > 1 else 2
data, n = W.paper_input(S, "int", seed=0, device="cuda")
k = data.clone()
ws = vm.Workspace()
vm.sort_(k, workspace=ws)
k.copy_(data)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); vm.sort_(k, workspace=ws); e1.record(); e1.synchronize()
print("n", n, "ms", e0.elapsed_time(e1))
