"""Python handle on the C++ MoE layer (libfsmoe.so, include/fsmoe_layer.h).

Torch allocates the parameters, gradients and activations (device memory and
streams are the only things torch provides); every FLOP of forward and
backward happens in the C++ executor and the sm_100a kernels behind it.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import torch

from . import _native as NL

GATE_KINDS = {"noisy_topk": 0, "sigmoid_topk": 1, "cosine_topk": 2, "expert_choice": 3}
FFN_KINDS = {"simple": 0, "gated3": 1}


class LayerConfigC(C.Structure):
    _fields_ = [
        ("tokens", C.c_int), ("model_dim", C.c_int), ("ffn_dim", C.c_int), ("experts", C.c_int),
        ("top_k", C.c_int), ("gate_kind", C.c_int), ("ffn_kind", C.c_int),
        ("capacity", C.c_longlong), ("proj_dim", C.c_int), ("seed", C.c_uint64),
        ("precision", C.c_int), ("r_fwd", C.c_int), ("r_bwd", C.c_int), ("device", C.c_int),
        ("dense_grad_elems", C.c_longlong), ("n_ar_slices", C.c_int),
        ("ar_slices", C.POINTER(C.c_longlong)), ("capacity_factor", C.c_double),
        ("unlimited", C.c_int), ("transport", C.c_int),
    ]


class LayerParamsC(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("w_gate", "w_noise", "proj", "w1", "w2", "g_gate",
                                          "g_noise", "g_proj", "g_w1", "g_w2", "dense_grad")]


@dataclass
class MoEConfig:
    tokens: int
    model_dim: int
    ffn_dim: int
    experts: int
    top_k: int = 1
    gate: str = "noisy_topk"
    ffn: str = "simple"
    capacity: int = 0            # 0 -> capacity_tokens(k, capacity_factor, unlimited)
    capacity_factor: float = 1.0
    unlimited: bool = False
    transport: str = ""          # "" (FSMOE_EP_TRANSPORT or peer), "peer", "ce", "nccl"
    proj_dim: int = 0
    seed: int = 7
    precision: str = "bf16"      # or "f32" (check mode)
    r_fwd: int = 1
    r_bwd: int = 1
    dense_grad_elems: int = 0
    ar_slices: list = field(default_factory=list)

    def resolved_capacity(self) -> int:
        """capacity_tokens (workload.cpp:43-51) with B*L = tokens (expert
        choice: tokens per expert, the same formula)."""
        if self.capacity:
            return self.capacity
        if self.unlimited:
            return self.top_k * self.tokens
        v = self.top_k * self.capacity_factor * self.tokens / self.experts
        return int(math.ceil(v - 1e-9))


def broadcast_unique_id(uid: bytes, world: int) -> bytes:
    """Rank 0's 128-byte NCCL unique id to every rank (torch.distributed is
    only the bootstrap channel; the data path is libfsmoe.so's own NCCL comm)."""
    import torch.distributed as dist
    if world <= 1 or not dist.is_initialized():
        return uid
    obj = [bytes(uid)]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


class EpGroup:
    """NCCL expert-parallel communicator owned by libfsmoe.so."""

    def __init__(self, world: int, rank: int, device: int, max_ctas: int = 0):
        lib = NL.cpp_lib()
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            NL.check(lib.fsmoe_ep_unique_id(uid), lib)
        uid = (C.c_ubyte * 128)(*broadcast_unique_id(bytes(uid), world))
        h = C.c_void_p()
        NL.check(lib.fsmoe_ep_create(world, rank, uid, device, max_ctas, C.byref(h)), lib)
        self.h = h
        self.world, self.rank = world, rank

    @classmethod
    def local_group(cls, world: int, device: int) -> list["EpGroup"]:
        """The single-GPU multi-rank harness (fsmoe_ep_create_local): `world`
        logical ranks of one group on one device, no NCCL / IPC. Create and
        drive each rank's MoELayer from its own thread (run_ranks)."""
        lib = NL.cpp_lib()
        hs = (C.c_void_p * world)()
        NL.check(lib.fsmoe_ep_create_local(world, device, hs), lib)
        out = []
        for r in range(world):
            g = cls.__new__(cls)
            g.h, g.world, g.rank = C.c_void_p(hs[r]), world, r
            out.append(g)
        return out

    def allreduce(self, t: torch.Tensor):
        """In-place sum of an fp32 / fp64 CUDA tensor over the group, on the
        current stream (fsmoe_ep_allreduce)."""
        assert t.is_cuda and t.is_contiguous() and t.dtype in (torch.float32, torch.float64)
        lib = NL.cpp_lib()
        NL.check(lib.fsmoe_ep_allreduce(self.h, C.c_void_p(t.data_ptr()), C.c_longlong(t.numel()),
                                        1 if t.dtype == torch.float64 else 0,
                                        C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)), lib)
        return t

    def close(self):
        if self.h:
            NL.cpp_lib().fsmoe_ep_destroy(self.h)
            self.h = None


def run_ranks(world: int, fn, timeout: float = 600.0):
    """Run fn(rank) for every logical rank of a local group on its own host
    thread (each with its own current CUDA stream) and return the results in
    rank order; the first exception is re-raised. ctypes drops the GIL in
    foreign calls, so the ranks' collectives (host barriers) meet."""
    import threading
    res, err = [None] * world, [None] * world

    def body(r):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                res[r] = fn(r)
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
        if t.is_alive():
            raise TimeoutError("local EP group: a rank did not finish")
    for e in err:
        if e is not None:
            raise e
    return res


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def gate_params(cfg: MoEConfig, init_seed: int):
    """Replicated gate parameters (fp64, identical on every rank)."""
    M, E = cfg.model_dim, cfg.experts
    g = torch.Generator(device="cpu").manual_seed(init_seed)
    rows = cfg.proj_dim if cfg.gate == "cosine_topk" else M
    w_gate = (torch.rand(rows, E, generator=g, dtype=torch.float64) * 2 - 1) / math.sqrt(rows)
    w_noise = (torch.rand(M, E, generator=g, dtype=torch.float64) * 2 - 1) / math.sqrt(M)
    proj = None
    if cfg.gate == "cosine_topk":
        proj = (torch.rand(cfg.proj_dim, M, generator=g, dtype=torch.float64) * 2 - 1) / math.sqrt(M)
    return w_gate, w_noise, proj


def expert_params(cfg: MoEConfig, rank: int, world: int, init_seed: int):
    """Rank-local expert weights [E_l][N1][M], [E_l][M][H] (fp32, CPU)."""
    M, H = cfg.model_dim, cfg.ffn_dim
    el = cfg.experts // world
    n1 = 2 * H if cfg.ffn == "gated3" else H
    ge = torch.Generator(device="cpu").manual_seed(init_seed * 1000 + 17 + rank)
    w1 = (torch.rand(el, n1, M, generator=ge) * 2 - 1) / math.sqrt(M)
    w2 = (torch.rand(el, M, H, generator=ge) * 2 - 1) / math.sqrt(H)
    return w1, w2


class MoELayer:
    """One FSMoE MoE layer on the current CUDA device (EP over `ep`)."""

    def __init__(self, cfg: MoEConfig, ep: EpGroup | None = None, device=None, init_seed=0):
        self.cfg = cfg
        self.ep = ep
        self.world = ep.world if ep else 1
        self.rank = ep.rank if ep else 0
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.device = dev
        assert cfg.experts % self.world == 0
        self.el = cfg.experts // self.world
        self.n1 = 2 * cfg.ffn_dim if cfg.ffn == "gated3" else cfg.ffn_dim
        self.act_dtype = torch.bfloat16 if cfg.precision == "bf16" else torch.float32
        M, H, E = cfg.model_dim, cfg.ffn_dim, cfg.experts
        # replicated gate parameters (same on every rank): fp64 master copies
        wg, wn, pj = gate_params(cfg, init_seed)
        self.w_gate, self.w_noise = wg.to(dev), wn.to(dev)
        self.proj = pj.to(dev) if pj is not None else None
        # rank-local experts (a different stream per rank)
        w1, w2 = expert_params(cfg, self.rank, self.world, init_seed)
        self.w1, self.w2 = w1.to(dev, self.act_dtype), w2.to(dev, self.act_dtype)
        self.g_gate = torch.zeros_like(self.w_gate)
        self.g_noise = torch.zeros_like(self.w_noise)
        self.g_proj = torch.zeros_like(self.proj) if self.proj is not None else None
        self.g_w1 = torch.zeros(self.el, self.n1, M, device=dev)
        self.g_w2 = torch.zeros(self.el, M, H, device=dev)
        self.dense_grad = (torch.zeros(cfg.dense_grad_elems, device=dev)
                           if cfg.dense_grad_elems else None)

        lib = NL.cpp_lib()
        c = LayerConfigC()
        c.tokens, c.model_dim, c.ffn_dim, c.experts = cfg.tokens, M, H, E
        c.top_k = cfg.top_k
        c.gate_kind = GATE_KINDS[cfg.gate]
        c.ffn_kind = FFN_KINDS[cfg.ffn]
        c.capacity = 0  # the C++ side derives it (capacity_tokens, workload.cpp:43-51)
        c.capacity_factor = cfg.capacity_factor
        c.unlimited = 1 if cfg.unlimited else 0
        c.transport = {"": 0, "peer": 1, "ce": 2, "nccl": 3}[cfg.transport]
        if cfg.capacity:
            c.capacity = cfg.capacity
        c.proj_dim = cfg.proj_dim
        c.seed = cfg.seed
        c.precision = 0 if cfg.precision == "bf16" else 1
        c.r_fwd, c.r_bwd = cfg.r_fwd, cfg.r_bwd
        c.device = dev.index
        c.dense_grad_elems = cfg.dense_grad_elems
        self._slices = (C.c_longlong * max(len(cfg.ar_slices), 1))(*cfg.ar_slices)
        c.n_ar_slices = len(cfg.ar_slices)
        c.ar_slices = C.cast(self._slices, C.POINTER(C.c_longlong))
        h = C.c_void_p()
        NL.check(lib.fsmoe_layer_create(C.byref(c), ep.h if ep else None, C.byref(h)), lib)
        self.h = h
        lib.fsmoe_layer_capacity.restype = C.c_longlong
        self.capacity = lib.fsmoe_layer_capacity(h)
        self.bind()

    def bind(self):
        lib = NL.cpp_lib()
        p = LayerParamsC()
        p.w_gate, p.w_noise, p.proj = _p(self.w_gate), _p(self.w_noise), _p(self.proj)
        p.w1, p.w2 = _p(self.w1), _p(self.w2)
        p.g_gate, p.g_noise, p.g_proj = _p(self.g_gate), _p(self.g_noise), _p(self.g_proj)
        p.g_w1, p.g_w2, p.dense_grad = _p(self.g_w1), _p(self.g_w2), _p(self.dense_grad)
        NL.check(lib.fsmoe_layer_bind(self.h, C.byref(p)), lib)

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def forward(self, x, y=None):
        assert x.is_cuda and x.dtype == self.act_dtype and x.shape == (self.cfg.tokens, self.cfg.model_dim)
        if y is None:
            y = torch.empty_like(x)
        lib = NL.cpp_lib()
        NL.check(lib.fsmoe_layer_forward(self.h, _p(x), _p(y), self._stream()), lib)
        self._x_saved = x  # the backward reads x (gate gradient): keep it alive
        return y

    def backward(self, dy, dx=None):
        if dx is None:
            dx = torch.empty_like(dy)
        lib = NL.cpp_lib()
        NL.check(lib.fsmoe_layer_backward(self.h, _p(dy), _p(dx), self._stream()), lib)
        return dx

    def set_trace(self, on: bool = True):
        """Record a measured per-phase timeline on both streams (synchronises)."""
        lib = NL.cpp_lib()
        NL.check(lib.fsmoe_layer_set_trace(self.h, 1 if on else 0), lib)

    def trace_json(self) -> str:
        """Chrome-trace JSON of the traced calls since set_trace(True)."""
        lib = NL.cpp_lib()
        lib.fsmoe_layer_trace.restype = C.c_longlong
        n = lib.fsmoe_layer_trace(self.h, None, 0)
        buf = C.create_string_buffer(n)
        lib.fsmoe_layer_trace(self.h, buf, n)
        return buf.value.decode()

    def buffer(self, name, dtype, shape=None):
        """View of a named internal device buffer (tests / inspection)."""
        lib = NL.cpp_lib()
        ptr, nbytes = C.c_void_p(), C.c_longlong()
        NL.check(lib.fsmoe_layer_buffer(self.h, name.encode(), C.byref(ptr), C.byref(nbytes)), lib)
        n = nbytes.value // torch.tensor([], dtype=dtype).element_size()
        out = torch.empty(n, dtype=dtype, device=self.device)
        if n:
            NL.check(NL.cuda_lib().fsmoe_copy_device(_p(out), ptr, C.c_size_t(nbytes.value),
                                                     self._stream()))
        return out if shape is None else out.view(shape)

    def close(self):
        if self.h:
            NL.cpp_lib().fsmoe_layer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
