"""Torch-tensor front end over the C ABI (include/fsmoe_cuda.h).

Torch supplies device memory and streams only; every op below is one call
into libfsmoe_cuda.so. Inputs must be CUDA tensors — there is no CPU path.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as NL

GATE_KINDS = {"noisy_topk": 0, "sigmoid_topk": 1, "cosine_topk": 2, "expert_choice": 3}
DTYPES = {torch.float64: 0, torch.float32: 1, torch.bfloat16: 2}
EPI = {"store_bf16": 0, "store_f32": 1, "gelu_fwd": 2, "swiglu_fwd": 3, "gelu_bwd": 4,
       "swiglu_bwd": 5}


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("fsmoe ops take CUDA tensors only (no CPU fallback)")
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def grouped_gemm(kind, A, B, D, *, nblk, rows, K=0, N=0, Mo=0, No=0, n_w=1, b_mn_major=False,
                 valid_rows=None, epi="store_bf16", D2=None, Zin=None, ldd=None, ldd2=0, ldz=0,
                 accumulate=False, precision=0):
    """Grouped expert GEMM (see csrc/gemm.h). kind: 'row' or 'k'."""
    lib = NL.cuda_lib()
    d = NL.GemmDesc()
    d.kind = 0 if kind == "row" else 1
    d.nblk, d.rows, d.K, d.N, d.Mo, d.No, d.n_w = nblk, rows, K, N, Mo, No, n_w
    d.b_mn_major = int(b_mn_major)
    d.A, d.B = _ptr(A), _ptr(B)
    d.valid_rows = _ptr(valid_rows)
    d.epi = EPI[epi] if isinstance(epi, str) else int(epi)
    d.D, d.D2, d.Zin = _ptr(D), _ptr(D2), _ptr(Zin)
    if ldd is None:
        ldd = N if kind == "row" else No
    d.ldd, d.ldd2, d.ldz = ldd, ldd2, ldz
    d.accumulate = int(accumulate)
    d.precision = precision
    NL.check(lib.fsmoe_grouped_gemm(C.byref(d), _stream()))


def activation_f32(op, rows, units, inp, z, out, out2=None):
    lib = NL.cuda_lib()
    NL.check(lib.fsmoe_activation_f32(EPI[op], C.c_longlong(rows), units, _ptr(inp), _ptr(z),
                                     _ptr(out), _ptr(out2), _stream()))
