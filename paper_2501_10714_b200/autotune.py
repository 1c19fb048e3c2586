"""On-box online profiling -> bench CSV -> fit_profile -> plan_layer: the
FSMoE loop that picks a layer's pipeline degrees from measured costs
(§5 "online profiling").

* Samples are (kind, n, t_ms) with the reference's kinds and units
  (json_io.cpp:262-300 bench CSV `kind,n,t_ms`; cost_models.cpp:61-125 fit):
  a2a / ag / rs / ar in elements moved per rank, gemm in the planner's
  MAC unit t*M*H (t = capacity per expert, workload.cpp:53-79 — the per-layer
  constant E_local*P is absorbed by the fitted slope).
* Collectives are timed with torch.distributed over NCCL (the library the
  executor's NCCL transport and gradient allreduces use); the GEMM with this
  package's tcgen05 grouped GEMM at the layer's own block shape.
* `plan()` feeds the fitted profile and the layer's task volumes to the
  bit-exact planner port (plan.py -> libfsmoe.so) and returns r_fwd / r_bwd.
"""
from __future__ import annotations

import csv
import io
import math

import numpy as np
import torch

from . import ops
from . import plan as P

KINDS = ("a2a", "ag", "rs", "ar", "gemm")


def write_bench_csv(samples, path=None) -> str:
    """The reference's bench CSV (json_io.cpp:262-300): header kind,n,t_ms."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(["kind", "n", "t_ms"])
    for k, n, t in samples:
        if k not in KINDS:
            raise ValueError(f"unknown kind '{k}'")
        w.writerow([k, repr(float(n)), repr(float(t))])
    text = buf.getvalue()
    if path:
        with open(path, "w") as f:
            f.write(text)
    return text


def read_bench_csv(text: str):
    """Parse with the reference's rules: exact header, 3 fields, known kinds."""
    lines = [ln.rstrip("\r") for ln in text.splitlines()]
    if not lines:
        raise ValueError("bench csv line 1: empty file")
    if lines[0].split(",") != ["kind", "n", "t_ms"]:
        raise ValueError("bench csv line 1: expected header kind,n,t_ms")
    out = []
    for i, ln in enumerate(lines[1:], start=2):
        if not ln:
            continue
        cells = ln.split(",")
        if len(cells) != 3:
            raise ValueError(f"bench csv line {i}: expected 3 fields, got {len(cells)}")
        if cells[0] not in KINDS:
            raise ValueError(f"bench csv line {i}: unknown kind '{cells[0]}'")
        out.append((cells[0], float(cells[1]), float(cells[2])))
    return out


def _time_ms(fn, reps=10, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def _max_over_ranks(v: float) -> float:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return v


def profile_collectives(sizes, dtype=torch.bfloat16, reps=10):
    """a2a / ag / rs / ar samples at `sizes` elements per rank (max over ranks).
    On one rank the collectives degenerate to local copies (what they cost)."""
    import torch.distributed as dist
    world = dist.get_world_size() if dist.is_initialized() else 1
    out = []
    for n in sizes:
        n = int(math.ceil(n / world) * world)
        x = torch.empty(n, dtype=dtype, device="cuda").normal_()
        y = torch.empty_like(x)
        xa = torch.empty(n, dtype=torch.float32, device="cuda").normal_()
        if world > 1:
            fns = {
                "a2a": lambda: dist.all_to_all_single(y, x),
                "ag": lambda: dist.all_gather_into_tensor(y, x[: n // world]),
                "rs": lambda: dist.reduce_scatter_tensor(y[: n // world], x),
                "ar": lambda: dist.all_reduce(xa),
            }
        else:
            fns = {"a2a": lambda: y.copy_(x), "ag": lambda: y.copy_(x), "rs": lambda: y.copy_(x),
                   "ar": lambda: xa.add_(0.0)}
        for k, fn in fns.items():
            if world > 1:
                dist.barrier()
            out.append((k, float(n), _max_over_ranks(_time_ms(fn, reps))))
    return out


def profile_gemm(nblk, caps, M, H, reps=10, unit_h=None):
    """Expert-GEMM samples: one grouped launch over the layer's nblk blocks of
    c rows (c in caps), K = M, N = H; n = c*M*unit_h (the planner's MAC unit,
    unit_h = hidden_scale * M; H by default)."""
    unit_h = unit_h or H
    out = []
    bf = torch.bfloat16
    for c in caps:
        X = torch.randn(nblk, c, M, device="cuda").to(bf)
        W = (torch.randn(nblk, H, M, device="cuda") / math.sqrt(M)).to(bf)
        Z = torch.empty(nblk, c, H, device="cuda", dtype=bf)
        fn = lambda: ops.grouped_gemm("row", X, W, Z, nblk=nblk, rows=c, K=M, N=H, n_w=nblk)  # noqa: E731
        out.append(("gemm", float(c) * M * unit_h, _max_over_ranks(_time_ms(fn, reps))))
    return out


def hidden_scale(cfg) -> int:
    """The reference's integer LayerConfig::hidden_scale (H = hidden_scale * M,
    workload.hpp:20) nearest to the layer's H / M (Mixtral: 14336 / 4096 = 3.5
    -> 4). The GEMM samples are recorded in the same planner unit
    (profile_gemm), so the fitted slope absorbs the difference."""
    return max(1, int(round(cfg.ffn_dim / cfg.model_dim)))


def layer_of(cfg) -> P.Layer:
    """MoEConfig -> the planner's LayerConfig (B = 1, L = local tokens)."""
    hs = hidden_scale(cfg)
    return P.Layer(batch=1, heads=1, seq_len=cfg.tokens, model_dim=cfg.model_dim, hidden_scale=hs,
                   capacity_factor=cfg.capacity_factor, ffn=cfg.ffn, experts=cfg.experts,
                   top_k=cfg.top_k)


def collect(cfg, world: int, reps=10, r_max=8):
    """Online profile for one layer shape on this box: collectives around the
    layer's a2a volume, and the GEMM at exactly the chunk sizes the planner
    chooses between (capacity C split into r = 1..r_max 128-row granule
    chunks, as the executor splits it): the fitted per-launch alpha then
    carries the wave quantisation of small chunks on 148 SMs, which a fit over
    a few far-apart sizes smooths away."""
    layer = layer_of(cfg)
    vol = P.derive_volumes(layer, (world, world, 1, 1, world, 1))
    a2a = vol[0]
    sizes = [a2a / 8, a2a / 4, a2a / 2, a2a]
    cap = int(vol[6])
    ng = max(1, -(-cap // 128))
    caps = sorted({max(128, (ng // r) * 128) for r in range(1, r_max + 1)})
    while len(caps) < 3:          # small capacities: the fit still needs a slope
        caps.append(caps[-1] * 2)
    return profile_collectives(sizes, reps=reps) + profile_gemm(
        cfg.experts, caps, cfg.model_dim, cfg.ffn_dim, reps=reps,
        unit_h=hidden_scale(cfg) * cfg.model_dim), vol


def plan(cfg, samples, world: int, r_max=8, t_gar_bwd_ms=0.0):
    """fit_profile -> plan_layer (bit-exact reference port). Returns the plan
    dict plus the profile and fit quality."""
    prof, min_r2, clamped = P.fit_profile(samples)
    vol = P.derive_volumes(layer_of(cfg), (world, world, 1, 1, world, 1))
    out = P.plan_layer(vol, prof, t_gar_bwd_ms=t_gar_bwd_ms, r_max=r_max)
    out.update(profile=[float(v) for v in prof], min_r2=float(min_r2), clamped_mask=clamped,
               volumes=[float(v) for v in vol])
    return out


def step_ms(layer, x, dy, steps=10, warmup=3):
    """Measured forward + backward of one layer (CUDA events, max over ranks)."""
    y, dx = torch.empty_like(x), torch.empty_like(x)
    for _ in range(warmup):
        layer.forward(x, y)
        layer.backward(dy, dx)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        layer.forward(x, y)
        layer.backward(dy, dx)
    e.record()
    torch.cuda.synchronize()
    return _max_over_ranks(s.elapsed_time(e) / steps)


def refine(cfg, ep, r_plan, x, dy, r_max=8, steps=10, transports=None):
    """Online check of a plan on the real layer (the paper's online
    profiling, closing the loop the analytic model leaves open): measure the
    step at the planned degree and its neighbours r-1, r+1 (both passes move
    together), keep the fastest. With `transports` (EP only) every candidate
    degree is tried on each transport ("peer" only at r = 1 and the plan's r:
    its dispatch does not pipeline). Returns (r_fwd, r_bwd, {key: ms}) with
    key = r, or (transport, r) when transports are given; cfg.transport is
    set to the winner's."""
    from .layer import MoELayer
    r0 = max(r_plan)
    rs = sorted({max(1, r0 - 1), r0, min(r_max, r0 + 1)})
    if transports:
        # the copy-engine pipeline needs r >= 2 to overlap anything: try 2 too
        ce_rs = sorted({r for r in rs + [2] if 2 <= r <= r_max})
        cand = [(t, r) for t in transports for r in (sorted({1, r0}) if t == "peer" else ce_rs)]
    else:
        cand = rs
    meas = {}
    keep = (cfg.r_fwd, cfg.r_bwd, cfg.transport)
    for c in cand:
        t, r = c if transports else (cfg.transport, c)
        cfg.r_fwd = cfg.r_bwd = r
        cfg.transport = t
        layer = MoELayer(cfg, ep, init_seed=1)
        meas[c] = step_ms(layer, x, dy, steps=steps)
        layer.close()
    cfg.r_fwd, cfg.r_bwd, cfg.transport = keep
    best = min(meas, key=meas.get)
    if transports:
        cfg.transport = best[0]
        return best[1], best[1], meas
    return best, best, meas


def autotune(cfg, world: int, reps=10, r_max=8):
    """Profile this box, plan, and return cfg with r_fwd / r_bwd set."""
    samples, _ = collect(cfg, world, reps=reps)
    p = plan(cfg, samples, world, r_max=r_max)
    cfg.r_fwd, cfg.r_bwd = p["r_fwd"], p["r_bwd"]
    return cfg, p, samples
