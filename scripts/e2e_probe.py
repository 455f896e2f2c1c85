"""End-to-end (pinned host buffers -> vmps_sort_pairs_host -> pinned host)
throughput of 2^30 cfg5 batches with NS rotating streams.
usage: python scripts/e2e_probe.py NS [batches]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27147_b200 as vm
import workloads as W
NS = int(sys.argv[1]); KB = int(sys.argv[2]) if len(sys.argv) > 2 else 9
dev = torch.device("cuda")
n = 1 << 30
k0, v0 = W.cfg5(n=n, device=dev)
hk = torch.empty(n, dtype=torch.int32, pin_memory=True).view(torch.uint32); hk.copy_(k0)
hv = torch.empty(n, dtype=torch.int32, pin_memory=True).view(torch.uint32); hv.copy_(v0)
del k0, v0
outs = [(torch.empty(n, dtype=torch.int32, pin_memory=True).view(torch.uint32),
         torch.empty(n, dtype=torch.int32, pin_memory=True).view(torch.uint32)) for _ in range(NS)]
streams = [torch.cuda.Stream(dev) for _ in range(NS)]
dbufs = [(torch.empty(n, dtype=torch.uint32, device=dev), torch.empty(n, dtype=torch.uint32, device=dev)) for _ in range(NS)]
wss = [vm.Workspace() for _ in range(NS)]
def step(q):
    j = q % NS
    vm.sort_host_(hk, hv, device=dev, out_keys=outs[j][0], out_values=outs[j][1], d_keys=dbufs[j][0],
                  d_values=dbufs[j][1], workspace=wss[j], stream=streams[j])
for q in range(NS): step(q)
torch.cuda.synchronize()
cur = torch.cuda.current_stream(dev)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(cur)
for s in streams: s.wait_event(e0)
for q in range(KB): step(q)
for s in streams:
    ev = torch.cuda.Event(); ev.record(s); cur.wait_event(ev)
e1.record(cur); e1.synchronize()
ms = e0.elapsed_time(e1) / KB
print(json.dumps({"NS": NS, "batches": KB, "ms_per_batch": ms, "gkeys_s": n / (ms / 1000) / 1e9}))
