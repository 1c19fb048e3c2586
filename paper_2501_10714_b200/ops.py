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
       "swiglu_bwd": 5, "add_bf16": 6}


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("fsmoe ops take CUDA tensors only (no CPU fallback)")
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


# tile-variant override for every grouped_gemm call (tests sweep the variants):
# (ctas, bn) with 0 = the library's heuristic
GEMM_FORCE = (0, 0)


def grouped_gemm(kind, A, B, D, *, nblk, rows, K=0, N=0, Mo=0, No=0, n_w=1, b_mn_major=False,
                 rows_total=0, row0=0, valid_rows=None, epi="store_bf16", D2=None, Zin=None, ldd=None, ldd2=0, ldz=0,
                 accumulate=False, precision=0, force=None, dbg=0, order=(0, 0), scatter_rows=None,
                 scatter_out=None):
    """Grouped expert GEMM (see csrc/gemm.h). kind: 'row' or 'k'. scatter_rows /
    scatter_out: output row r goes to row scatter_rows[r] of scatter_out (< 0 dropped)."""
    lib = NL.cuda_lib()
    d = NL.GemmDesc()
    d.kind = 0 if kind == "row" else 1
    d.nblk, d.rows, d.K, d.N, d.Mo, d.No, d.n_w = nblk, rows, K, N, Mo, No, n_w
    d.rows_total, d.row0 = rows_total, row0
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
    d.force_ctas, d.force_bn = force if force is not None else GEMM_FORCE
    d.dbg = dbg
    d.band_m, d.band_n = order
    if scatter_rows is not None:
        d.scatter_rows, d.scatter_out = _ptr(scatter_rows), _ptr(scatter_out)
        d.scatter_ld = scatter_out.shape[-1]
    NL.check(lib.fsmoe_grouped_gemm(C.byref(d), _stream()))


def activation_f32(op, nblk, rows_total, row0, rows, units, inp, z, out):
    lib = NL.cuda_lib()
    NL.check(lib.fsmoe_activation_f32(EPI[op], nblk, rows_total, row0, rows, units, _ptr(inp),
                                     _ptr(z), _ptr(out), _stream()))


# ----------------------------------------------------------------- routing --

def _i(t):
    return _ptr(t)


def _ws(nbytes, device):
    return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def gate_desc(kind, top_k, seed, x, w_score, w_noise=None, proj=None):
    d = NL.GateDesc()
    d.kind = GATE_KINDS[kind] if isinstance(kind, str) else int(kind)
    d.top_k = int(top_k)
    d.seed = int(seed) & (2 ** 64 - 1)
    d.tokens, d.model_dim = (x.shape[0], x.shape[1]) if x.dim() == 2 else (0, 0)
    d.x_dtype = DTYPES[x.dtype]
    d.score_rows, d.score_cols = w_score.shape
    if w_noise is not None:
        d.noise_rows, d.noise_cols = w_noise.shape
    if proj is not None:
        d.proj_rows, d.proj_cols = proj.shape
    return d


def gate(kind, top_k, seed, x, w_score, w_noise=None, proj=None, save=False, check=True):
    """fsmoe::run_gate (workload.cpp:143-235) on the GPU. Returns
    (pick_token, pick_expert, pick_weight[, saved dict])."""
    lib = NL.cuda_lib()
    d = gate_desc(kind, top_k, seed, x, w_score, w_noise, proj)
    NL.check(lib.fsmoe_gate_validate(C.byref(d)))
    dev = x.device
    T, E = d.tokens, d.score_cols
    n = T * d.top_k if d.kind != 3 else E * d.top_k
    tok = torch.empty(n, dtype=torch.int32, device=dev)
    exp = torch.empty(n, dtype=torch.int32, device=dev)
    w = torch.empty(n, dtype=torch.float64, device=dev)
    saved = {}
    if save:
        saved["scores"] = torch.empty(T * E, dtype=torch.float64, device=dev)
        if d.kind == 0:
            saved["noise"] = torch.empty(T * E, dtype=torch.float64, device=dev)
            saved["spread"] = torch.empty(T * E, dtype=torch.float64, device=dev)
        if d.kind == 2:
            saved["proj"] = torch.empty(T * d.proj_rows, dtype=torch.float64, device=dev)
    status = torch.zeros(2, dtype=torch.int32, device=dev)
    lib.fsmoe_gate_workspace_size.restype = C.c_size_t
    wsb = lib.fsmoe_gate_workspace_size(C.byref(d))
    ws = _ws(wsb, dev)
    NL.check(lib.fsmoe_gate(C.byref(d), _ptr(x), _ptr(w_score), _ptr(w_noise), _ptr(proj),
                            _i(tok), _i(exp), _ptr(w), _ptr(saved.get("scores")),
                            _ptr(saved.get("noise")), _ptr(saved.get("spread")),
                            _ptr(saved.get("proj")), _i(status), _ptr(ws), C.c_size_t(wsb),
                            _stream()))
    if check:
        NL.check(lib.fsmoe_check_status(_i(status), _stream()))
    if save:
        return tok, exp, w, saved
    return tok, exp, w


def assign(pick_token, pick_expert, tokens, experts, capacity, check=True):
    """Capacity assignment of dispatch_tokens (workload.cpp:248-262)."""
    lib = NL.cuda_lib()
    dev = pick_token.device
    P = pick_token.numel()
    slot = torch.empty(max(P, 1), dtype=torch.int32, device=dev)
    fill = torch.empty(max(experts, 1), dtype=torch.int64, device=dev)
    dropped = torch.empty(1, dtype=torch.int64, device=dev)
    pos = torch.empty(max(experts * max(capacity, 0), 1), dtype=torch.int32, device=dev)
    status = torch.zeros(2, dtype=torch.int32, device=dev)
    lib.fsmoe_assign_workspace_size.restype = C.c_size_t
    wsb = lib.fsmoe_assign_workspace_size(C.c_longlong(P), experts)
    ws = _ws(wsb, dev)
    NL.check(lib.fsmoe_assign(C.c_longlong(P), _i(pick_token), _i(pick_expert), tokens, experts,
                              C.c_longlong(capacity), _i(slot), _i(fill), _i(dropped), _i(pos),
                              _i(status), _ptr(ws), C.c_size_t(wsb), _stream()))
    if check:
        NL.check(lib.fsmoe_check_status(_i(status), _stream()))
    return slot[:P], fill[:experts], dropped, pos[:experts * capacity]


def token_index(pick_token, tokens, token_major_k=0):
    lib = NL.cuda_lib()
    dev = pick_token.device
    P = pick_token.numel()
    ptr = torch.empty(tokens + 1, dtype=torch.int32, device=dev)
    idx = torch.empty(max(P, 1), dtype=torch.int32, device=dev)
    lib.fsmoe_token_index_workspace_size.restype = C.c_size_t
    wsb = lib.fsmoe_token_index_workspace_size(C.c_longlong(P), tokens)
    ws = _ws(wsb, dev)
    NL.check(lib.fsmoe_token_index(C.c_longlong(P), _i(pick_token), tokens, token_major_k,
                                   _i(ptr), _i(idx), _ptr(ws), C.c_size_t(wsb), _stream()))
    return ptr, idx[:P]


def slot_row(slot, experts, capacity, chunks):
    lib = NL.cuda_lib()
    lib.fsmoe_slot_row.restype = C.c_longlong
    return lib.fsmoe_slot_row(C.c_longlong(slot), experts, C.c_longlong(capacity), chunks)


def dispatch(x, pick_of_slot, pick_token, experts, capacity, chunks=1, out=None):
    """Order: buffers[(experts*capacity) x M] (chunk-major when chunks > 1)."""
    lib = NL.cuda_lib()
    M = x.shape[1]
    if out is None:
        out = torch.empty(experts * capacity, M, dtype=x.dtype, device=x.device)
    NL.check(lib.fsmoe_dispatch(DTYPES[x.dtype], M, experts, C.c_longlong(capacity), chunks,
                                _i(pick_of_slot), _i(pick_token), _ptr(x), _ptr(out), _stream()))
    return out


def gather_rows(src, src_row, out=None):
    """out[i] = src[src_row[i]] (src_row < 0: zero row), TMA row moves."""
    lib = NL.cuda_lib()
    n, M = src_row.numel(), src.shape[1]
    if out is None:
        out = torch.empty(n, M, dtype=src.dtype, device=src.device)
    NL.check(lib.fsmoe_gather_rows(DTYPES[src.dtype], M, C.c_longlong(n), _i(src_row), _ptr(src),
                                   _ptr(out), None, _stream()))
    return out


def peer_map(bases, rank, experts_local, capacity):
    m = NL.PeerRows()
    for i, b in enumerate(bases):
        m.base[i] = b.data_ptr() if torch.is_tensor(b) else b
    m.world, m.rank, m.experts_local, m.capacity = len(bases), rank, experts_local, capacity
    return m


def dispatch_peer(x, pick_of_slot, pick_token, experts, capacity, dst_map):
    lib = NL.cuda_lib()
    NL.check(lib.fsmoe_dispatch_peer(DTYPES[x.dtype], x.shape[1], experts, C.c_longlong(capacity),
                                     _i(pick_of_slot), _i(pick_token), _ptr(x), C.byref(dst_map),
                                     _stream()))


def peer_signal(flags, slot):
    NL.check(NL.cuda_lib().fsmoe_peer_signal(C.byref(flags), slot, None, C.c_longlong(0), None,
                                             _stream()))


def peer_wait(flags, slot, target):
    NL.check(NL.cuda_lib().fsmoe_peer_wait(C.byref(flags), slot, C.c_ulonglong(target), _stream()))


def combine(buffers, tok_ptr, tok_pick, slot_of_pick, pick_weight, tokens, experts, capacity,
            chunks=1, out=None):
    """I-Order: y[t] = sum_{kept picks} w * buffers[slot] (workload.cpp:266-282)."""
    lib = NL.cuda_lib()
    M = buffers.shape[1]
    if out is None:
        out = torch.empty(tokens, M, dtype=buffers.dtype, device=buffers.device)
    NL.check(lib.fsmoe_combine(DTYPES[buffers.dtype], tokens, M, experts, C.c_longlong(capacity),
                               chunks, _i(tok_ptr), _i(tok_pick), _i(slot_of_pick),
                               _ptr(pick_weight), _ptr(buffers), _ptr(out), _stream()))
    return out


def combine_bwd(dy, buffers, pick_of_slot, pick_token, pick_weight, experts, capacity, chunks=1):
    lib = NL.cuda_lib()
    T, M = dy.shape
    P = pick_token.numel()
    dbuf = torch.empty_like(buffers)
    dw = torch.empty(max(P, 1), dtype=torch.float64, device=dy.device)
    NL.check(lib.fsmoe_combine_bwd(DTYPES[dy.dtype], T, M, experts, C.c_longlong(capacity), chunks,
                                   C.c_longlong(P), _i(pick_of_slot), _i(pick_token),
                                   _ptr(pick_weight), None, _ptr(dy), _ptr(buffers), _ptr(dbuf),
                                   _ptr(dw), _stream()))
    return dbuf, dw[:P]


def dispatch_bwd(dbuf, tok_ptr, tok_pick, slot_of_pick, tokens, experts, capacity, chunks=1,
                 dx=None, accumulate=False):
    lib = NL.cuda_lib()
    M = dbuf.shape[1]
    if dx is None:
        dx = torch.empty(tokens, M, dtype=dbuf.dtype, device=dbuf.device)
    NL.check(lib.fsmoe_dispatch_bwd(DTYPES[dbuf.dtype], tokens, M, experts, C.c_longlong(capacity),
                                    chunks, _i(tok_ptr), _i(tok_pick), _i(slot_of_pick),
                                    _ptr(dbuf), _ptr(dx), int(accumulate), _stream()))
    return dx


def gate_bwd(kind, top_k, seed, x, w_score, w_noise, proj, pick_token, pick_expert, pick_weight,
             d_weight, saved, dx, d_w_score, d_w_noise=None, d_proj=None):
    """Accumulates gate parameter grads (fp64) and dx (x dtype)."""
    lib = NL.cuda_lib()
    d = gate_desc(kind, top_k, seed, x, w_score, w_noise, proj)
    lib.fsmoe_gate_bwd_workspace_size.restype = C.c_size_t
    wsb = lib.fsmoe_gate_bwd_workspace_size(C.byref(d))
    ws = _ws(wsb, x.device)
    NL.check(lib.fsmoe_gate_bwd(C.byref(d), _ptr(x), _ptr(w_score), _ptr(w_noise), _ptr(proj),
                                _i(pick_token), _i(pick_expert), _ptr(pick_weight),
                                _ptr(d_weight), _ptr(saved.get("scores")),
                                _ptr(saved.get("noise")), _ptr(saved.get("spread")),
                                _ptr(saved.get("proj")), _ptr(dx), _ptr(d_w_score),
                                _ptr(d_w_noise), _ptr(d_proj), _ptr(ws), C.c_size_t(wsb),
                                _stream()))
