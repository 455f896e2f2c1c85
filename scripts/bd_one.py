"""One scratch-bounded sort of a cfg5-shaped input (n = 2^LOG2N, cap
4 sqrt(n log2 n), cells per VMPS_BD_CELL or one piece) for ncu captures of
the bounded kernels."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27147_b200 as vm
import workloads as W
lg = int(os.environ.get("LOG2N", "28"))
n = 1 << lg
k0, v0 = W.cfg5(n=n, device="cuda")
S = int(4 * math.sqrt(n * math.log2(n)))
cell = int(os.environ.get("VMPS_BD_CELL", "0"))
if cell:
    vm.lib().vmps_test_set_bd_chunk(cell)
k, v = k0.clone(), v0.clone()
vm.sort_(k, v, scratch=S)
torch.cuda.synchronize()
ku, vu = k0.clone(), v0.clone()
vm.sort_(ku, vu)
print("equal_unbounded", bool(torch.equal(ku, k) and torch.equal(vu, v)))
