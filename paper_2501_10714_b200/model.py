"""A stack of MoE layers whose backward executes the FSMoE gradient-partition
plan (grad_partition.cpp:185-228, §5): the
replicated dense gradients of every layer form one pool in backward order,
and each layer's MoE backward synchronises a contiguous run of the pool —
gradient produced by layers that already finished their backward, oldest
first — in its inter-link slot between the last dispatch and the first
combine AlltoAll (schedule_sim.cpp:185-188), on the layer's comm stream,
overlapping the expert GEMMs. What no window absorbs is synchronised after
the last layer (the tail).

The dense blocks themselves (attention etc.) are outside this framework: a
layer's dense gradient is handed in by the caller (`produce`) and the plan
runs with t_olp_dense = 0, so every assignment rides an MoE slot.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import autotune
from . import plan as P
from .layer import MoEConfig, MoELayer


def _parse_plan(out, n):
    rows = out[: 9 * n].reshape(n, 9)
    keys = ("n_first", "n_first_dense", "n_first_moe", "x_g", "t_gar_ms", "degree", "case",
            "t_olp_moe_ms", "t_olp_dense_ms")
    layers = [dict(zip(keys, map(float, r))) for r in rows]
    tail = dict(tail_elements=float(out[9 * n]), tail_ms=float(out[9 * n + 1]),
                objective_ms=float(out[9 * n + 2]), step2_ran=bool(out[9 * n + 3]))
    return layers, tail


def slot_loads(plan_layers, n_grad: int, n_layers: int):
    """Integer elements each layer's slot synchronises, by rounding the plan's
    cumulative (conserved) counts; also checks availability: layer i may only
    sync gradient produced by layers < i."""
    cum, out = 0.0, []
    prev = 0
    for i, a in enumerate(plan_layers):
        cum += a["n_first"] + a["x_g"]
        c = int(round(cum))
        c = min(c, i * n_grad)  # availability (plan guarantees it up to rounding)
        out.append(max(c - prev, 0))
        prev = max(prev, c)
    tail = n_layers * n_grad - prev
    return out, tail


class MoEStack:
    """n_layers identical MoE layers (own weights) on this rank's GPU, EP over
    `ep`; `plan_profile` = a fitted profile (plan.fit_profile) or None to
    profile this box (autotune.collect)."""

    def __init__(self, cfg: MoEConfig, n_layers: int, ep=None, n_grad: int | None = None,
                 plan_profile=None, sync="plan", de=(0, 200, 0.8, 0.9, 1)):
        self.cfg, self.L, self.ep = cfg, n_layers, ep
        self.world = ep.world if ep else 1
        self.n_grad = n_grad if n_grad is not None else 4 * cfg.model_dim * cfg.model_dim
        layer = autotune.layer_of(cfg)
        par = (self.world, self.world, 1, 1, self.world, 1)
        vol = P.derive_volumes(layer, par)
        if plan_profile is None:
            samples, _ = autotune.collect(cfg, self.world)
            plan_profile = P.fit_profile(samples)[0]
        self.profile = plan_profile
        out = P.build_partition_plan([(vol, 0.0, float(self.n_grad))] * n_layers, plan_profile, de)
        self.plan_layers, self.plan_tail = _parse_plan(out, n_layers)
        if sync == "plan":
            self.loads, self.tail = slot_loads(self.plan_layers, self.n_grad, n_layers)
        elif sync == "tail":  # everything after the backward (the non-overlapped baseline)
            self.loads, self.tail = [0] * n_layers, n_layers * self.n_grad
        else:
            raise ValueError(sync)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.pool = torch.zeros(n_layers * self.n_grad, dtype=torch.float32, device=dev)
        self.layers = []
        for i in range(n_layers):
            # layers[i] is the i-th in FORWARD order; its backward position is L-1-i
            j = n_layers - 1 - i
            c = MoEConfig(**{**cfg.__dict__})
            c.dense_grad_elems = max(self.loads[j], 0)
            c.ar_slices = [self.loads[j]] if self.loads[j] > 0 else []
            self.layers.append(MoELayer(c, ep, init_seed=1 + i))
        self._acts = []

    def forward(self, x):
        self._acts = [x]
        for l in self.layers:
            x = l.forward(x)
            self._acts.append(x)
        return x

    def backward(self, dy, produce=None):
        """produce(j, segment): fills backward-position j's dense gradient (the
        caller's dense block); default leaves the pool as it is."""
        ptr = 0
        for j, l in enumerate(reversed(self.layers)):
            n = self.loads[j]
            if n > 0:
                # this layer's slot syncs pool[ptr, ptr + n): gradient of layers < j
                l.dense_grad = self.pool[ptr: ptr + n]
                l.bind()
            dy = l.backward(dy)
            ptr += n
            if produce is not None:
                produce(j, self.pool[j * self.n_grad: (j + 1) * self.n_grad])
        if self.world > 1 and ptr < self.pool.numel():
            # the tail, over the layers' own EP communicator (libfsmoe.so)
            self.ep.allreduce(self.pool[ptr:])
        return dy

    def close(self):
        for l in self.layers:
            l.close()
