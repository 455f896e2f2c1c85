import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_27147_b200 as vm
import workloads as W
from tests.test_gpu_parity import _structured
rng = np.random.default_rng(200)
vm.test_set_tiles(64, 16, 0)
for trial in range(40):
    n = int(rng.integers(2, 6000))
    keys = _structured(rng, n, np.uint32)
    mr = int(rng.choice([0, 1, 2, 3, 16]))
    vm.test_set_minrun(mr)
    k = W.from_numpy(keys, 'cuda'); v = torch.arange(n, dtype=torch.int32, device='cuda').view(torch.uint32)
    print('trial', trial, 'n', n, 'minrun', mr, flush=True)
    vm.sort_(k, v)
    torch.cuda.synchronize()
    ko = np.sort(keys, kind='stable')
    assert (W.to_numpy(k) == ko).all(), 'mismatch'
print('ok')
