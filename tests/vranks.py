"""Test helper: run a function on g virtual ranks of the native multi-GPU
protocol -- g threads of this process on one GPU, each with its own CUDA
stream and a communicator of one vmps_local_group (csrc/comm.cu).  ctypes
releases the GIL inside library calls, so the ranks run concurrently."""
from __future__ import annotations

import os
import threading

import torch


def run(g: int, fn, device: int = 0, timeout: float = 600.0):
    """fn(rank, comm) on every rank (inside torch.cuda.stream(own stream));
    returns the results in rank order; re-raises the first failure."""
    import paper_2605_27147_b200 as vm
    os.environ.setdefault("VMPS_COMM_TIMEOUT_S", "120")  # a stuck test fails instead of hanging
    group = vm.LocalGroup(g, device)
    comms = [vm.Comm.local(r, group) for r in range(g)]
    out = [None] * g
    err = [None] * g

    def body(r):
        try:
            torch.cuda.set_device(device)
            s = torch.cuda.Stream(device)
            with torch.cuda.stream(s):
                out[r] = fn(r, comms[r])
            s.synchronize()
        except BaseException as e:  # noqa: BLE001 -- reported below
            err[r] = e

    ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(g)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    alive = any(t.is_alive() for t in ts)
    for c in comms:
        c.destroy()
    if not alive:
        group.destroy()
    assert not alive, "a virtual rank did not finish"
    for e in err:
        if e is not None:
            raise e
    return out
