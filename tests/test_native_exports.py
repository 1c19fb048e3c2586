"""The drop-in boundary loads without a GPU and exports every entry point its
headers declare (include/fsmoe_cuda.h, include/fsmoe_layer.h,
include/fsmoe_plan.h); host-only entry points answer without a device.
CPU only."""
import ctypes as C
import os
import re

import pytest

from paper_2501_10714_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fsmoe_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header,lib", [("fsmoe_cuda.h", "cuda"), ("fsmoe_layer.h", "cpp"),
                                        ("fsmoe_plan.h", "cpp")])
def test_every_declared_symbol_is_exported(header, lib):
    so = _native.cuda_lib() if lib == "cuda" else _native.cpp_lib()
    names = declared(header)
    assert len(names) >= 5
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing


def test_host_entry_points_without_gpu():
    lib = _native.cuda_lib()
    assert lib.fsmoe_abi_version() == 1
    lib.fsmoe_slot_row.restype = C.c_longlong
    # chunk-major slot map is a permutation (host arithmetic only)
    E, Cap, r = 3, 10, 3
    rows = sorted(lib.fsmoe_slot_row(C.c_longlong(s), E, C.c_longlong(Cap), r) for s in range(E * Cap))
    assert rows == list(range(E * Cap))
    # validation errors are raised before any device work, with the reference's text
    from paper_2501_10714_b200 import ops
    d = _native.GateDesc()
    d.kind, d.top_k, d.tokens, d.model_dim, d.score_rows, d.score_cols = 1, 3, 4, 8, 8, 2
    rc = lib.fsmoe_gate_validate(C.byref(d))
    assert rc == 2 and lib.fsmoe_last_error() == b"gate: top_k exceeds expert count"
    assert ops.GATE_KINDS["expert_choice"] == 3


def test_ops_refuse_cpu_tensors():
    import torch
    from paper_2501_10714_b200 import ops
    x = torch.zeros(4, 8, dtype=torch.float64)
    with pytest.raises(ValueError, match="CUDA tensors only"):
        ops.dispatch(x, x, x, 2, 2)
