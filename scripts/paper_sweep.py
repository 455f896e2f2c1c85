"""The paper's own workload sweep on one B200:
N = 10^7 (n ~ U[9N/10, N], general non-power-of-two n), values uniform in
[100, 10^9], pre-sorted runs of length Geom(1/S), S in {2, 1e2, ..., 1e6}, for
the paper's data types: int (u32 keys), randomBlob30 and zeroBlob30 (120-byte
records, lexicographic), ptr (the permutation of randomBlob30 records only).
One JSON line per (type, S): ms per sort (CUDA events, median of 5 after 2
warm-ups, input restored untimed), Mkeys/s, and for int the plan statistics.
usage: python scripts/paper_sweep.py [out.jsonl]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_27147_b200 as vm
import workloads as W

out = open(sys.argv[1], "w") if len(sys.argv) > 1 else sys.stdout
dev = torch.device("cuda")
ws = vm.Workspace()


def timed(fn, restore, reps=5, warm=2):
    for _ in range(warm):
        restore(); fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        restore()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


for kind in ("int", "randomBlob30", "zeroBlob30", "ptr"):
    for S in W.PAPER_S:
        data, n = W.paper_input(S, "randomBlob30" if kind == "ptr" else kind, seed=0, device=dev)
        rec = {"type": kind, "S": S, "n": n}
        if kind == "int":
            k = data.clone()
            st = vm.sort_(k, stats=True, workspace=ws)
            ok = bool(torch.equal(k.view(torch.int32).to(torch.int64) & 0xFFFFFFFF,
                                  torch.sort(data.view(torch.int32).to(torch.int64) & 0xFFFFFFFF).values))
            ms = timed(lambda: vm.sort_(k, workspace=ws), lambda: k.copy_(data))
            rec.update(runs=st["runs"], M_over_n=st["merge_cost_M"] / n, minrun=st["minrun"], verified=ok)
        else:
            r = data.view(torch.int32)
            o = torch.empty_like(r)
            perm_only = kind == "ptr"

            def fn():
                if perm_only:
                    vm.sort_records(r, out=o, perm=True, workspace=ws)  # records_out is written too
                else:
                    vm.sort_records(r, out=o, workspace=ws)
            fn()
            torch.cuda.synchronize()
            # full verification: permutation, records_out = records[perm],
            # stable lexicographic order over all 30 words
            _, pm = vm.sort_records(r, perm=True, workspace=ws)
            torch.cuda.synchronize()
            p64 = pm.to(torch.int64) & 0xFFFFFFFF
            a = o.to(torch.int64) & 0xFFFFFFFF
            diff = a[1:] != a[:-1]
            anyd = diff.any(dim=1)
            first = torch.argmax(diff.to(torch.int32), dim=1)
            rows = torch.arange(a.shape[0] - 1, device=a.device)
            ok = (bool((torch.bincount(p64, minlength=n) == 1).all()) and torch.equal(o, r[p64])
                  and bool(((~anyd) | (a[1:][rows, first] > a[:-1][rows, first])).all())
                  and bool((anyd | (p64[1:] > p64[:-1])).all()))
            del a, diff, anyd, first, rows, p64
            ms = timed(fn, lambda: None)
            rec.update(record_bytes=120, verified=ok)
        rec.update(ms=ms, mkeys_per_s=n / (ms / 1000) / 1e6)
        print(json.dumps(rec), file=out, flush=True)
