"""Python front end over the host control plane of libfsmoe.so
(include/fsmoe_plan.h): capacity / task volumes, alpha-beta profile fit,
pipeline-degree optimizer, schedule simulator and gradient partitioner — the
FSMoE planner that sets the executor's r_fwd / r_bwd and allreduce slices."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as NL

KINDS = {"a2a": 0, "ag": 1, "rs": 2, "ar": 3, "gemm": 4}
STYLES = {"fsmoe": 0, "fsmoe_no_iio": 1, "pipemoe": 2, "sequential": 3}


def _lib():
    lib = NL.cpp_lib()
    lib.fsmoe_capacity_tokens.restype = C.c_longlong
    return lib


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(C.POINTER(C.c_int))


def _check(rc):
    NL.check(rc, NL.cpp_lib())


@dataclass
class Layer:
    """LayerConfig (workload.hpp:13-26)."""
    batch: int
    heads: int
    seq_len: int
    model_dim: int
    hidden_scale: int
    capacity_factor: float = 1.0
    unlimited: bool = False
    ffn: str = "simple"
    experts: int = 8
    top_k: int = 1
    t_olp_dense_ms: float = 0.0
    grad_override: float | None = None

    def arrays(self):
        ints = [self.batch, self.heads, self.seq_len, self.model_dim, self.hidden_scale,
                int(self.unlimited), int(self.ffn == "gated3"), self.experts, self.top_k,
                int(self.grad_override is not None)]
        dbls = [self.capacity_factor, self.t_olp_dense_ms, self.grad_override or 0.0]
        return ints, dbls


def capacity_tokens(layer: Layer) -> int:
    ints, dbls = layer.arrays()
    ia, ip = _i(ints)
    da, dp = _d(dbls)
    lib = _lib()
    v = lib.fsmoe_capacity_tokens(ip, dp)
    if v < 0:
        NL.check(2, lib)
    return int(v)


def derive_volumes(layer: Layer, parallel) -> np.ndarray:
    """[a2a, ag, rs, gemm_macs, gemm_count, grad, capacity]; parallel = (total_gpus,
    gpus_per_node, dp, tp, ep, esp)."""
    ints, dbls = layer.arrays()
    (ia, ip), (da, dp), (pa, pp) = _i(ints), _d(dbls), _i(list(parallel))
    out, op = _d(np.zeros(7))
    _check(_lib().fsmoe_derive_volumes(ip, dp, pp, op))
    return out


def pipeline_chunks(capacity: int, r: int):
    out = np.zeros(2 * max(r, 1), dtype=np.int32)
    n = _lib().fsmoe_pipeline_chunks(C.c_longlong(capacity), r, out.ctypes.data_as(C.POINTER(C.c_int)))
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(n)]


def fit_profile(samples, min_r2=0.0):
    """samples: iterable of (kind, n, t_ms). Returns (profile[10], min_r2, clamped_mask)."""
    kinds = [KINDS.get(k, 99) for k, _, _ in samples]
    (ka, kp) = _i(kinds)
    (na, np_) = _d([s[1] for s in samples])
    (ta, tp) = _d([s[2] for s in samples])
    prof, pp = _d(np.zeros(10))
    meta, mp = _d(np.zeros(2))
    _check(_lib().fsmoe_fit_profile(len(kinds), kp, np_, tp, C.c_double(min_r2), pp, mp))
    return prof, meta[0], int(meta[1])


def find_degree(volumes, profile, t_gar_ms=0.0, exp_multiplier=1, r_max=16):
    (va, vp), (pa, pp) = _d(volumes), _d(profile)
    out, op = _d(np.zeros(11))
    _check(_lib().fsmoe_find_degree(vp, pp, C.c_double(t_gar_ms), exp_multiplier, r_max, op))
    return out


def plan_layer(volumes, profile, t_gar_bwd_ms=0.0, r_max=16):
    (va, vp), (pa, pp) = _d(volumes), _d(profile)
    out, op = _d(np.zeros(10))
    _check(_lib().fsmoe_plan_layer(vp, pp, C.c_double(t_gar_bwd_ms), r_max, op))
    return dict(r_fwd=int(out[0]), case_fwd=int(out[1]), t_moe_fwd_ms=out[2],
                boundary_fwd=bool(out[3]), r_bwd=int(out[4]), case_bwd=int(out[5]),
                t_moe_bwd_ms=out[6], boundary_bwd=bool(out[7]), t_gar_bwd_ms=out[8],
                t_olp_moe_bwd_ms=out[9])


def build_partition_plan(layers, profile, de=(0, 200, 0.8, 0.9, 1), r_max=16):
    """layers: list of (volumes[7], t_olp_dense_ms, n_grad)."""
    flat = np.concatenate([np.concatenate([np.asarray(v, float), [d, g]]) for v, d, g in layers])
    (la, lp), (pa, pp), (da, dp) = _d(flat), _d(profile), _d(de)
    n = len(layers)
    out, op = _d(np.zeros(9 * n + 4))
    _check(_lib().fsmoe_build_partition_plan(n, lp, pp, dp, r_max, op))
    return out


def simulate_stage(volumes, profile, exp_multiplier, r, sync_ms=(), style="fsmoe"):
    (va, vp), (pa, pp), (sa, sp) = _d(volumes), _d(profile), _d(list(sync_ms) or [0.0])
    cap = 5 + 2 * (5 * r + len(sync_ms) + 8)
    out, op = _d(np.zeros(cap))
    _check(_lib().fsmoe_simulate_stage(vp, pp, exp_multiplier, r, len(sync_ms), sp,
                                       STYLES[style], op, cap))
    return out


def brute_force_degree(volumes, profile, t_gar_ms=0.0, exp_multiplier=1, r_max=16):
    (va, vp), (pa, pp) = _d(volumes), _d(profile)
    out, op = _d(np.zeros(2))
    _check(_lib().fsmoe_brute_force_degree(vp, pp, C.c_double(t_gar_ms), exp_multiplier, r_max, op))
    return int(out[0]), out[1]
