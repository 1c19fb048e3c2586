"""ctypes bindings to the in-tree native libraries.

libfsmoe_cuda.so (include/fsmoe_cuda.h) holds every sm_100a kernel of the
path; libfsmoe.so (include/fsmoe/*.hpp) the C++ drop-in and MoE layer. There
is no CPU fallback: if the libraries are missing this module raises on import
of any op, and the ops refuse CPU tensors.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "lib")
CUDA_SO = os.path.join(LIB_DIR, "libfsmoe_cuda.so")
CPP_SO = os.path.join(LIB_DIR, "libfsmoe.so")

_cuda = None
_cpp = None


class NativeError(RuntimeError):
    """Raised with the library's fsmoe_last_error() text."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class ConfigError(NativeError):
    """Mirror of fsmoe::ConfigError (common.hpp:16-18), status 2."""


class FitQualityError(NativeError):
    """Mirror of fsmoe::FitQualityError (common.hpp:22-24), status 3."""


class InvariantError(NativeError):
    """Mirror of fsmoe::InvariantError (common.hpp:26-28), status 4."""


class GemmDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("nblk", C.c_int), ("rows", C.c_int), ("K", C.c_int),
        ("N", C.c_int), ("Mo", C.c_int), ("No", C.c_int), ("n_w", C.c_int),
        ("rows_total", C.c_int), ("row0", C.c_int), ("b_mn_major", C.c_int), ("A", C.c_void_p), ("B", C.c_void_p),
        ("valid_rows", C.c_void_p), ("epi", C.c_int), ("D", C.c_void_p), ("D2", C.c_void_p),
        ("Zin", C.c_void_p), ("ldd", C.c_longlong), ("ldd2", C.c_longlong),
        ("ldz", C.c_longlong), ("accumulate", C.c_int), ("precision", C.c_int),
        ("d_peers", C.c_void_p), ("blk_lo", C.c_int), ("blk_hi", C.c_int), ("blk_exclude", C.c_int),
        ("max_sms", C.c_int), ("force_ctas", C.c_int), ("force_bn", C.c_int), ("dbg", C.c_int),
        ("band_m", C.c_int), ("band_n", C.c_int),
        ("scatter_rows", C.c_void_p), ("scatter_out", C.c_void_p), ("scatter_ld", C.c_longlong),
    ]


class PeerRows(C.Structure):
    """fsmoe_peer_rows (include/fsmoe_cuda.h): where rows of a [P][E_l][C]
    block buffer land (identity for one rank)."""
    _fields_ = [("base", C.c_void_p * 8), ("world", C.c_int), ("rank", C.c_int),
                ("experts_local", C.c_int), ("capacity", C.c_longlong)]


class PeerFlags(C.Structure):
    """fsmoe_peer_flags: per-rank uint64 arrival counters [nslots][world]."""
    _fields_ = [("base", C.c_void_p * 8), ("world", C.c_int), ("rank", C.c_int),
                ("nslots", C.c_int), ("wait_ns", C.c_void_p), ("timeout_ns", C.c_ulonglong)]


class GateDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("top_k", C.c_int), ("seed", C.c_uint64), ("tokens", C.c_int),
        ("model_dim", C.c_int), ("x_dtype", C.c_int), ("score_rows", C.c_int),
        ("score_cols", C.c_int), ("noise_rows", C.c_int), ("noise_cols", C.c_int),
        ("proj_rows", C.c_int), ("proj_cols", C.c_int),
    ]


def cuda_lib() -> C.CDLL:
    global _cuda
    if _cuda is None:
        if not os.path.exists(CUDA_SO):
            raise ImportError(f"{CUDA_SO} missing: build with __graft_entry__.build() "
                              "(there is no CPU fallback)")
        _cuda = C.CDLL(CUDA_SO)
        _cuda.fsmoe_last_error.restype = C.c_char_p
    return _cuda


def cpp_lib() -> C.CDLL:
    global _cpp
    if _cpp is None:
        cuda_lib()
        if not os.path.exists(CPP_SO):
            raise ImportError(f"{CPP_SO} missing: build with __graft_entry__.build()")
        _cpp = C.CDLL(CPP_SO)
        _cpp.fsmoe_layer_last_error.restype = C.c_char_p
    return _cpp


def check(rc: int, lib: C.CDLL | None = None) -> None:
    if rc == 0:
        return
    lib = lib or cuda_lib()
    # libfsmoe.so keeps its own message slot (it also re-exports the CUDA
    # library's symbols through its dependency, so test by identity).
    fn = lib.fsmoe_layer_last_error if lib is _cpp else lib.fsmoe_last_error
    fn.restype = C.c_char_p
    msg = (fn() or b"").decode()
    if rc == 2:
        raise ConfigError(rc, msg)
    if rc == 3:
        raise FitQualityError(rc, msg)
    if rc == 4:
        raise InvariantError(rc, msg)
    raise NativeError(rc, msg or f"native status {rc}")
