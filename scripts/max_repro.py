"""Repro for the maximum-size keys-only sort (run with VMPS_DEBUG_SYNC=1 to
name the failing kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27147_b200 as vm
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_maxsize import _fill, _check_sorted
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 32) - 37
k = _fill(n, 32, torch.device("cuda"))
try:
    st = vm.sort_(k, stats=True)
    torch.cuda.synchronize()
    print("ok", st["runs"], st["levels_executed"])
    _check_sorted(k)
    print("sorted ok")
except Exception as e:
    print("ERR", e)
