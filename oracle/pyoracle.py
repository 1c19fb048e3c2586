"""TEST INFRASTRUCTURE ONLY — ctypes front end for the CPU checkers.

Two interchangeable backends with the same call signatures:

* ``Oracle("port")``      -> oracle/lib/libfsmoe_oracle.so, the plain-C
  restatement of /root/reference/proj/src/workload.cpp (always available;
  built by ``make -C oracle oracle``).
* ``Oracle("reference")`` -> oracle/_ref/libfsmoe_ref.so, the reference's own
  sources compiled here (``make -C oracle ref``); absent on machines without
  /root/reference unless the built .so travelled with the tree.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline /
--impl reference) import this module. The product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "lib", "libfsmoe_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfsmoe_ref.so")

GATE_KINDS = {"noisy_topk": 0, "sigmoid_topk": 1, "cosine_topk": 2, "expert_choice": 3}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


@dataclass
class GateOut:
    token: np.ndarray
    expert: np.ndarray
    weight: np.ndarray


@dataclass
class DispatchOut:
    buffers: np.ndarray
    slot_of_pick: np.ndarray
    fill: np.ndarray
    dropped: int


def available(kind: str) -> bool:
    return os.path.exists(PORT_SO if kind == "port" else REF_SO)


def _mat(a, rows=None, cols=None):
    if a is None:
        return np.zeros((0, 0), dtype=np.float64)
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library not built: {path} (make -C oracle)")
        self.lib = C.CDLL(path)
        pre = "orc_" if kind == "port" else "ref_"
        self._gate = getattr(self.lib, pre + "run_gate")
        self._gate.restype = C.c_int
        self._gate.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, _dp,
                               C.c_int, C.c_int, _dp, C.c_int, C.c_int, _dp,
                               C.c_int, C.c_int, _dp, _ip, _ip, _dp,
                               C.POINTER(C.c_longlong), C.c_char_p, C.c_int]
        self._disp = getattr(self.lib, pre + "dispatch")
        self._disp.restype = C.c_int
        self._disp.argtypes = [C.c_int, C.c_int, _dp, C.c_int, C.c_longlong, _ip, _ip,
                               C.c_longlong, _dp, _ip, _lp, C.POINTER(C.c_longlong),
                               C.c_char_p, C.c_int]
        self._comb = getattr(self.lib, pre + "combine")
        self._comb.restype = C.c_int
        if kind == "port":
            self._comb.argtypes = [C.c_int, C.c_int, _dp, C.c_int, C.c_longlong, _ip, _dp,
                                   C.c_longlong, _ip, C.c_int, _dp, C.c_char_p, C.c_int]
        else:
            self._comb.argtypes = [C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_longlong,
                                   _ip, _ip, _dp, C.c_longlong, _ip, C.c_int, _dp,
                                   C.c_char_p, C.c_int]

    # -- run_gate (workload.cpp:143-235) ---------------------------------
    def run_gate(self, kind, top_k, seed, x, w_score, w_noise=None, proj=None) -> GateOut:
        x = _mat(x)
        ws, wn, pj = _mat(w_score), _mat(w_noise), _mat(proj)
        T, M = x.shape
        E = ws.shape[1] if ws.ndim == 2 else 0
        cap = max(T * max(top_k, 0), E * max(top_k, 0), 1)
        tok = np.zeros(cap, np.int32)
        exp = np.zeros(cap, np.int32)
        w = np.zeros(cap, np.float64)
        n = C.c_longlong(0)
        err = C.create_string_buffer(256)
        k = GATE_KINDS[kind] if isinstance(kind, str) else int(kind)
        rc = self._gate(k, int(top_k), C.c_uint64(int(seed) & (2**64 - 1)), T, M,
                        x if x.size else np.zeros(1), ws.shape[0], ws.shape[1],
                        ws if ws.size else np.zeros(1), wn.shape[0], wn.shape[1],
                        wn if wn.size else np.zeros(1), pj.shape[0], pj.shape[1],
                        pj if pj.size else np.zeros(1), tok, exp, w, C.byref(n), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        m = n.value
        return GateOut(tok[:m].copy(), exp[:m].copy(), w[:m].copy())

    # -- dispatch_tokens (workload.cpp:237-264) ---------------------------
    def dispatch(self, x, experts, pick_token, pick_expert, capacity) -> DispatchOut:
        x = _mat(x)
        T, M = x.shape
        pt = np.ascontiguousarray(pick_token, np.int32)
        pe = np.ascontiguousarray(pick_expert, np.int32)
        P = pt.size
        cap_ok = capacity if capacity > 0 else 0
        buf = np.zeros(max(experts * cap_ok * M, 1), np.float64)
        slot = np.zeros(max(P, 1), np.int32)
        fill = np.zeros(max(experts, 1), np.int64)
        dropped = C.c_longlong(0)
        err = C.create_string_buffer(256)
        rc = self._disp(T, M, x if x.size else np.zeros(1), experts, P,
                        pt if P else np.zeros(1, np.int32), pe if P else np.zeros(1, np.int32),
                        int(capacity), buf, slot, fill, C.byref(dropped), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return DispatchOut(buf[: experts * cap_ok * M].reshape(experts * cap_ok, M),
                           slot[:P].copy(), fill[:experts].copy(), dropped.value)

    # -- combine_tokens (workload.cpp:266-282) ----------------------------
    def combine(self, buffers, tokens, experts, pick_token, pick_expert, pick_weight,
                slot_of_pick, model_dim):
        b = _mat(buffers)
        pt = np.ascontiguousarray(pick_token, np.int32)
        pe = np.ascontiguousarray(pick_expert, np.int32)
        pw = np.ascontiguousarray(pick_weight, np.float64)
        sp = np.ascontiguousarray(slot_of_pick, np.int32)
        y = np.zeros(max(tokens * model_dim, 1), np.float64)
        err = C.create_string_buffer(256)
        one_i = np.zeros(1, np.int32)
        if self.kind == "port":
            rc = self._comb(b.shape[0], b.shape[1], b if b.size else np.zeros(1), tokens,
                            pt.size, pt if pt.size else one_i, pw if pw.size else np.zeros(1),
                            sp.size, sp if sp.size else one_i, model_dim, y, err, 256)
        else:
            rc = self._comb(b.shape[0], b.shape[1], b if b.size else np.zeros(1), tokens,
                            experts, pt.size, pt if pt.size else one_i,
                            pe if pe.size else one_i, pw if pw.size else np.zeros(1),
                            sp.size, sp if sp.size else one_i, model_dim, y, err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return y[: tokens * model_dim].reshape(tokens, model_dim)


# ------------------------------------------------------------------ helpers --

def mt_uniform_stream(seed: int):
    """Generator of the reference tests' 53-bit uniforms (test_util.hpp:92-96),
    computed through the C port's mt19937_64 so Python never re-derives it."""
    lib = C.CDLL(PORT_SO)

    class MT(C.Structure):
        _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]

    lib.orc_mt64_seed.argtypes = [C.POINTER(MT), C.c_uint64]
    lib.orc_mt64_next.argtypes = [C.POINTER(MT)]
    lib.orc_mt64_next.restype = C.c_uint64
    lib.orc_uniform_fill.argtypes = [C.POINTER(MT), C.c_longlong, C.c_double, C.c_double,
                                     C.POINTER(C.c_double)]
    g = MT()
    lib.orc_mt64_seed(C.byref(g), C.c_uint64(seed))
    return lib, g


class MtRng:
    """std::mt19937_64 draws (via the C port) + the reference's uniform()."""

    def __init__(self, seed: int):
        self.lib, self.g = mt_uniform_stream(seed)

    def next(self) -> int:
        return int(self.lib.orc_mt64_next(C.byref(self.g)))

    def uniform_array(self, n: int, lo: float, hi: float) -> np.ndarray:
        out = np.empty(max(n, 1), np.float64)
        self.lib.orc_uniform_fill(C.byref(self.g), C.c_longlong(n), C.c_double(lo),
                                  C.c_double(hi), out.ctypes.data_as(C.POINTER(C.c_double)))
        return out[:n]

    def matrix(self, rows: int, cols: int, lo: float, hi: float) -> np.ndarray:
        return self.uniform_array(rows * cols, lo, hi).reshape(rows, cols)


# --------------------------------------------------------------- planner --

class RefPlanner:
    """The reference's control plane (cost_models / pipeline_optimizer /
    schedule_sim / grad_partition), compiled from /root/reference by
    oracle/Makefile, behind the same flat-array calls as include/fsmoe_plan.h."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"reference not built: {REF_SO} (make -C oracle ref)")
        self.lib = C.CDLL(REF_SO)
        self.lib.ref_capacity_tokens.restype = C.c_longlong

    @staticmethod
    def _d(a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        return a, a.ctypes.data_as(C.POINTER(C.c_double))

    @staticmethod
    def _i(a):
        a = np.ascontiguousarray(a, dtype=np.int32)
        return a, a.ctypes.data_as(C.POINTER(C.c_int))

    def _call(self, name, *args):
        err = C.create_string_buffer(256)
        rc = getattr(self.lib, name)(*args, err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())

    def capacity_tokens(self, ints, dbls):
        (ia, ip), (da, dp) = self._i(ints), self._d(dbls)
        err = C.create_string_buffer(256)
        v = self.lib.ref_capacity_tokens(ip, dp, err, 256)
        if v < 0:
            raise OracleError(2, err.value.decode())
        return int(v)

    def derive_volumes(self, ints, dbls, parallel):
        (ia, ip), (da, dp), (pa, pp) = self._i(ints), self._d(dbls), self._i(parallel)
        out, op = self._d(np.zeros(7))
        self._call("ref_derive_volumes", ip, dp, pp, op)
        return out

    def fit_profile(self, kinds, ns, ts, min_r2):
        (ka, kp), (na, np_), (ta, tp) = self._i(kinds), self._d(ns), self._d(ts)
        prof, pp = self._d(np.zeros(10))
        meta, mp = self._d(np.zeros(2))
        self._call("ref_fit_profile", len(kinds), kp, np_, tp, C.c_double(min_r2), pp, mp)
        return prof, meta[0], int(meta[1])

    def find_degree(self, vol, prof, t_gar, mult, r_max):
        (va, vp), (pa, pp) = self._d(vol), self._d(prof)
        out, op = self._d(np.zeros(11))
        self._call("ref_find_degree", vp, pp, C.c_double(t_gar), mult, r_max, op)
        return out

    def plan_layer(self, vol, prof, t_gar, r_max):
        (va, vp), (pa, pp) = self._d(vol), self._d(prof)
        out, op = self._d(np.zeros(10))
        self._call("ref_plan_layer", vp, pp, C.c_double(t_gar), r_max, op)
        return out

    def build_partition_plan(self, layers_flat, n, prof, de, r_max):
        (la, lp), (pa, pp), (da, dp) = self._d(layers_flat), self._d(prof), self._d(de)
        out, op = self._d(np.zeros(9 * n + 4))
        self._call("ref_build_partition_plan", n, lp, pp, dp, r_max, op)
        return out

    def simulate_stage(self, vol, prof, mult, r, sync, style):
        (va, vp), (pa, pp), (sa, sp) = self._d(vol), self._d(prof), self._d(list(sync) or [0.0])
        cap = 5 + 2 * (5 * r + len(sync) + 8)
        out, op = self._d(np.zeros(cap))
        self._call("ref_simulate_stage", vp, pp, mult, r, len(sync), sp, style, op, cap)
        return out

    def brute_force_degree(self, vol, prof, t_gar, mult, r_max):
        (va, vp), (pa, pp) = self._d(vol), self._d(prof)
        out, op = self._d(np.zeros(2))
        self._call("ref_brute_force_degree", vp, pp, C.c_double(t_gar), mult, r_max, op)
        return int(out[0]), out[1]
