"""CPU-side checks of the boundary: libvmps.so loads without a GPU and exports
every function include/vmps.h declares; the product package never imports
the oracle; calls fail loudly (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "vmps.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vmps_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_2605_27147_b200 import build
    lib_path = build.build()
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib_path], text=True)
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    declared = header_functions()
    assert declared, "no functions parsed from include/vmps.h"
    missing = [f for f in declared if f not in exported]
    assert not missing, f"declared but not exported: {missing}"
    import paper_2605_27147_b200 as vm
    assert set(vm.EXPORTS) == set(declared)
    ctypes.CDLL(lib_path)  # loads on a CPU-only host


def test_workspace_query_without_gpu():
    import paper_2605_27147_b200 as vm
    n = 1 << 20
    nb = vm.workspace_bytes(n, vm.KEY_U32, 1)
    assert nb >= n * 8  # at least the ping-pong scratch of keys + payload
    assert vm.workspace_bytes(n, vm.KEY_U32, 0) < nb
    with pytest.raises(vm.VmpsError):
        vm.workspace_bytes(1 << 33, vm.KEY_U32, 1)
    assert vm.lib().vmps_status_string(3) == b"workspace or scratch budget too small"


def test_no_cpu_fallback():
    import torch
    import paper_2605_27147_b200 as vm
    with pytest.raises(ValueError):
        vm.sort_(torch.arange(10, dtype=torch.int32).view(torch.uint32))


def test_product_does_not_touch_oracle():
    pkg = os.path.join(ROOT, "paper_2605_27147_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).replace("oracle/", ""), f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".c", ".h", ".py")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(import|from)\s+paper_2605_27147_b200", txt, re.M), f
            assert "#include \"vmps.h\"" not in txt and "include/vmps.h" not in txt, f
