"""A stack of MoE layers whose backward executes the FSMoE gradient-partition
plan (grad_partition.cpp:185-228, §5): the
replicated dense gradients of every layer form one pool in backward order,
and each layer synchronises contiguous runs of the pool — gradient produced
by layers that already finished their backward, oldest first — in its two
windows:

* the MoE window: inside the layer's MoE backward, between the last
  dispatch and the first combine AlltoAll (schedule_sim.cpp:185-188), on the
  layer's comm stream, overlapping the expert GEMMs (n_first_moe + x_g);
* the dense window (`dense=True`): while the layer's dense block computes
  its backward, a pre-sync allreduce on a comm stream (the pre_sync tasks of
  build_backward_model_dag, schedule_sim.cpp:383-434; n_first_dense).

What no window absorbs is synchronised after the last layer (the tail).

With `dense=True` every layer has a dense block after its MoE layer (so its
backward runs first, as in the reference's backward model):
a chain of bf16 M x M projections (4 M^2 parameters, derive_volumes'
dense gradient, workload.cpp:53-79) run through torch / cuBLAS — it stands
for the attention block the framework does not own. Its measured backward
time is the plan's t_olp_dense. Without it the caller's `produce` fills
each layer's gradient and t_olp_dense = 0, so every assignment rides an MoE
window.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import autotune
from . import plan as P
from .layer import MoEConfig, MoELayer


class DenseBlock:
    """x -> x W_0^T W_1^T ... W_{k-1}^T (bf16, cuBLAS), k = n_grad / M^2; the
    backward writes the fp32 weight gradient into a caller-owned slice."""

    def __init__(self, M: int, n_grad: int, device, seed: int):
        k = max(1, n_grad // (M * M))
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.W = [((torch.rand(M, M, generator=g) * 2 - 1) / math.sqrt(M)).to(device, torch.bfloat16)
                  for _ in range(k)]
        self.n_grad = k * M * M
        self._h = []

    def forward(self, x):
        self._h = [x]
        for w in self.W:
            x = x @ w.T
            self._h.append(x)
        return x

    def backward(self, dy, grad_out):
        """grad_out: fp32 tensor of n_grad elements (this layer's pool slot)."""
        M = self.W[0].shape[0]
        gv = grad_out.view(len(self.W), M, M)
        for i in reversed(range(len(self.W))):
            gv[i].copy_(dy.T @ self._h[i])
            dy = dy @ self.W[i]
        return dy


def _parse_plan(out, n):
    rows = out[: 9 * n].reshape(n, 9)
    keys = ("n_first", "n_first_dense", "n_first_moe", "x_g", "t_gar_ms", "degree", "case",
            "t_olp_moe_ms", "t_olp_dense_ms")
    layers = [dict(zip(keys, map(float, r))) for r in rows]
    tail = dict(tail_elements=float(out[9 * n]), tail_ms=float(out[9 * n + 1]),
                objective_ms=float(out[9 * n + 2]), step2_ran=bool(out[9 * n + 3]))
    return layers, tail


def slot_loads(plan_layers, n_grad: int, n_layers: int):
    """Integer elements each backward position synchronises in its dense
    window (n_first_dense) and its MoE window (n_first_moe + x_g), by
    rounding the plan's cumulative (conserved) counts. Availability follows
    the reference's backward model (build_backward_model_dag: a layer's dense
    compute, which produces its gradient, precedes its MoE stage): the dense
    window of position i syncs only gradient of positions < i (step 1), the
    MoE window also position i's own (step 2's repair allows origins <= i).
    Returns (moe loads, dense loads, tail)."""
    cum, prev = 0.0, 0
    moe, dense = [], []
    for i, a in enumerate(plan_layers):
        for part, out, avail in ((a["n_first_dense"], dense, i * n_grad),
                                 (a["n_first_moe"] + a["x_g"], moe, (i + 1) * n_grad)):
            cum += part
            c = min(int(round(cum)), avail)  # (the plan guarantees it up to rounding)
            out.append(max(c - prev, 0))
            prev = max(prev, c)
    tail = n_layers * n_grad - prev
    return moe, dense, tail


class MoEStack:
    """n_layers identical MoE layers (own weights) on this rank's GPU, EP over
    `ep`; `plan_profile` = a fitted profile (plan.fit_profile) or None to
    profile this box (autotune.collect). `dense=True` puts a DenseBlock after
    every MoE layer and uses its measured backward time as the plan's dense
    window."""

    def __init__(self, cfg: MoEConfig, n_layers: int, ep=None, n_grad: int | None = None,
                 plan_profile=None, sync="plan", de=(0, 200, 0.8, 0.9, 1), dense=False,
                 t_olp_dense_ms=None):
        self.cfg, self.L, self.ep = cfg, n_layers, ep
        self.world = ep.world if ep else 1
        self.n_grad = n_grad if n_grad is not None else 4 * cfg.model_dim * cfg.model_dim
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dense = [DenseBlock(cfg.model_dim, self.n_grad, dev, 100 + i) for i in range(n_layers)] \
            if dense else None
        if self.dense:
            self.n_grad = self.dense[0].n_grad
            if t_olp_dense_ms is None:
                t_olp_dense_ms = self._time_dense_backward()
        self.t_olp_dense_ms = float(t_olp_dense_ms or 0.0)
        layer = autotune.layer_of(cfg)
        par = (self.world, self.world, 1, 1, self.world, 1)
        vol = P.derive_volumes(layer, par)
        if plan_profile is None:
            samples, _ = autotune.collect(cfg, self.world)
            plan_profile = P.fit_profile(samples)[0]
        self.profile = plan_profile
        out = P.build_partition_plan([(vol, self.t_olp_dense_ms, float(self.n_grad))] * n_layers,
                                     plan_profile, de)
        self.plan_layers, self.plan_tail = _parse_plan(out, n_layers)
        if sync == "plan":
            self.loads, self.dense_loads, self.tail = slot_loads(self.plan_layers, self.n_grad, n_layers)
        elif sync == "tail":  # everything after the backward (the non-overlapped baseline)
            self.loads, self.dense_loads = [0] * n_layers, [0] * n_layers
            self.tail = n_layers * self.n_grad
        elif sync == "none":  # measurement only: no gradient sync at all (the lower bound)
            self.loads, self.dense_loads, self.tail = [0] * n_layers, [0] * n_layers, 0
        else:
            raise ValueError(sync)
        self.pool = torch.zeros(n_layers * self.n_grad, dtype=torch.float32, device=dev)
        self.layers = []
        for i in range(n_layers):
            # layers[i] is the i-th in FORWARD order; its backward position is L-1-i
            j = n_layers - 1 - i
            c = MoEConfig(**{**cfg.__dict__})
            c.dense_grad_elems = max(self.loads[j], 0)
            c.ar_slices = [self.loads[j]] if self.loads[j] > 0 else []
            self.layers.append(MoELayer(c, ep, init_seed=1 + i))
        self.comm = torch.cuda.Stream(device=dev)
        self._acts = []

    def _time_dense_backward(self, reps=5):
        blk = self.dense[0]
        T, M = self.cfg.tokens, self.cfg.model_dim
        x = torch.randn(T, M, device=blk.W[0].device).to(torch.bfloat16)
        g = torch.empty(blk.n_grad, device=blk.W[0].device)
        blk.forward(x)
        for _ in range(2):
            blk.backward(x, g)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            blk.backward(x, g)
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps

    def forward(self, x):
        # block i: MoE layer, then its dense block — so the backward runs the
        # dense block first (producing the block's gradient) and the MoE stage
        # after it, the reference's per-layer backward order
        self._acts = [x]
        for i, l in enumerate(self.layers):
            x = l.forward(x)
            if self.dense:
                x = self.dense[i].forward(x)
            self._acts.append(x)
        return x

    def backward(self, dy, produce=None):
        """Backward in reverse layer order. produce(j, segment) fills
        backward-position j's dense gradient when there is no dense block
        (default: leave the pool as it is)."""
        ptr = 0
        cur = torch.cuda.current_stream()
        for j, l in enumerate(reversed(self.layers)):
            own = self.pool[j * self.n_grad: (j + 1) * self.n_grad]
            if self.dense:
                nd = self.dense_loads[j]
                if nd > 0 and self.world > 1:
                    # dense window: pre-sync older gradient (positions < j)
                    # beside this position's dense backward
                    self.comm.wait_stream(cur)
                    with torch.cuda.stream(self.comm):
                        self.ep.allreduce(self.pool[ptr: ptr + nd])
                ptr += nd
                dy = self.dense[self.L - 1 - j].backward(dy, own)
                # the pre-sync rides beside the dense backward only: it must be
                # done before the MoE backward issues its own collectives on
                # the same communicator (one NCCL op at a time, in issue order)
                cur.wait_stream(self.comm)
            elif produce is not None:
                produce(j, own)
            n = self.loads[j]
            if n > 0:
                # MoE window: pool[ptr, ptr + n) (positions <= j), inside the
                # MoE backward between its last dispatch and first combine
                l.dense_grad = self.pool[ptr: ptr + n]
                l.bind()
            dy = l.backward(dy)
            ptr += n
        cur.wait_stream(self.comm)
        if self.world > 1 and self.tail > 0 and ptr < self.pool.numel():
            # the tail, over the layers' own EP communicator (libfsmoe.so)
            self.ep.allreduce(self.pool[ptr:])
        return dy

    def close(self):
        for l in self.layers:
            l.close()
