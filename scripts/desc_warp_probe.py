"""One sort of cfg2 (2^24 random runs) for profiling the small-level
partition kernels (k4_desc_warp / k4_desc)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27147_b200 as vm
import workloads as W
k, v = W.make(2, device="cuda")
vm.sort_(k, v)
torch.cuda.synchronize()
