"""Expert parallelism on ONE GPU: the single-GPU multi-rank harness
(fsmoe_ep_create_local, include/fsmoe_layer.h).

P logical ranks share one device, each driven from its own host thread with
its own MoELayer, exactly as P processes drive P GPUs. The default
(peer-memory) transport runs unchanged: the dispatch kernel, the I-order
backward and the fwd2 / dgrad1 GEMM epilogues store their rows straight into
the owning rank's receive buffers and raise its arrival flags; only the
pointer exchange and the gate / dense gradient allreduces are replaced (host
barriers + an in-order summation kernel instead of CUDA IPC and NCCL).

Every rank's y, dx and expert / gate gradients are compared with the fp64
restatement (oracle/layer_oracle.py) applied per rank
with the union of experts — the same check tests/test_ep_gpu.py makes across
real GPUs (per-rank routing with local capacity) — plus: a
repeated step is bit-identical, replicated gradients carry the same bits on
every rank, and every rank's stream really waited on its peers' flags.
"""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(world, precision, gate, ffn, rf, rb, k=2, dense=0, split=None, T=1024, M=256, H=256,
         transport=None, experts_per_rank=None):
    import layer_oracle
    import pyoracle
    from paper_2501_10714_b200.layer import EpGroup, MoEConfig, MoELayer, expert_params, gate_params, run_ranks

    E = 4 * world if gate != "expert_choice" else 2 * world
    if experts_per_rank:
        E = experts_per_rank * world
    slices = [dense // 3, dense // 3, dense - 2 * (dense // 3)] if dense else []
    cfg = MoEConfig(tokens=T, model_dim=M, ffn_dim=H, experts=E, top_k=k, gate=gate, ffn=ffn,
                    precision=precision, seed=9, r_fwd=rf, r_bwd=rb,
                    capacity=384 if gate != "expert_choice" else 0,
                    proj_dim=16 if gate == "cosine_topk" else 0, dense_grad_elems=dense,
                    ar_slices=slices)
    dt = torch.bfloat16 if precision == "bf16" else torch.float32

    def inputs(r):
        g = torch.Generator().manual_seed(500 + r)
        return (torch.rand(T, M, generator=g) * 2 - 1).to(dt), (torch.rand(T, M, generator=g) * 2 - 1).to(dt)

    def dense_of(r):
        g = torch.Generator().manual_seed(900 + r)
        return torch.rand(dense, generator=g) * 2 - 1

    env = {}
    if split is not None:
        env["FSMOE_EP_SPLIT"] = str(split)
    if transport is not None:
        env["FSMOE_EP_TRANSPORT"] = transport
    old = {k_: os.environ.get(k_) for k_ in env}
    os.environ.update(env)
    try:
        groups = EpGroup.local_group(world, torch.cuda.current_device())
        layers = [None] * world

        def make(r):
            layers[r] = MoELayer(cfg, groups[r], init_seed=2)
            return layers[r].capacity

        caps = run_ranks(world, make)
    finally:
        for k_, v_ in old.items():
            if v_ is None:
                os.environ.pop(k_, None)
            else:
                os.environ[k_] = v_

    def step(r):
        L = layers[r]
        x, dy = inputs(r)
        if dense:
            L.dense_grad.copy_(dense_of(r))
        y = L.forward(x.cuda())
        dx = L.backward(dy.cuda())
        out = {"y": y.clone(), "dx": dx.clone(), "g_w1": L.g_w1.clone(), "g_w2": L.g_w2.clone(),
               "g_gate": L.g_gate.clone()}
        if dense:
            out["dense"] = L.dense_grad.clone()
        wait = L.buffer("wait_ns", torch.int64)
        out["wait_ns"] = int(wait.item())
        return out

    try:
        first = run_ranks(world, step)
        again = run_ranks(world, step)
    finally:
        run_ranks(world, lambda r: layers[r].close())
        for g in groups:
            g.close()

    for r in range(world):
        for key in first[r]:
            if key == "wait_ns":
                continue
            assert torch.equal(first[r][key], again[r][key]), f"rank {r}: repeated step differs in {key}"
        assert again[r]["wait_ns"] >= first[r]["wait_ns"] > 0  # it waited on peers at least once

    # fp64 restatement with the union of experts (rank-major), per rank
    C = caps[0]
    W1 = np.concatenate([expert_params(cfg, r, world, 2)[0].to(dt).double().numpy() for r in range(world)])
    W2 = np.concatenate([expert_params(cfg, r, world, 2)[1].to(dt).double().numpy() for r in range(world)])
    wg, wn, pj = (t.numpy() if t is not None else None for t in gate_params(cfg, 2))
    orc = pyoracle.Oracle("port")
    kk = C if gate == "expert_choice" else k
    sums, per = {}, []
    for r in range(world):
        xr, dyr = inputs(r)
        yr, cache = layer_oracle.forward(xr.double().numpy(), gate, kk, 9, C, wg, wn, pj, W1, W2, ffn, orc)
        gr = layer_oracle.backward(cache, dyr.double().numpy(), gate, kk, C, wg, wn, pj, W1, W2, ffn)
        for key in ("g_w1", "g_w2", "g_gate"):
            sums[key] = sums.get(key, 0) + gr[key]
        per.append((yr, gr))
    tol = 1e-4 if precision == "f32" else 3e-2

    def rel(a, b):
        a = a.double().cpu().numpy() if torch.is_tensor(a) else a
        return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))

    el = E // world
    bad = {}
    for r in range(world):
        o = first[r]
        errs = {"y": rel(o["y"], per[r][0]), "dx": rel(o["dx"], per[r][1]["dx"]),
                "g_w1": rel(o["g_w1"], sums["g_w1"][r * el:(r + 1) * el]),
                "g_w2": rel(o["g_w2"], sums["g_w2"][r * el:(r + 1) * el])}
        if np.abs(sums["g_gate"]).max() > 0:
            errs["g_gate"] = rel(o["g_gate"], sums["g_gate"])
        for a, b in errs.items():
            if not b < tol:
                bad[(r, a)] = b
        if dense:
            # the dense gradient: every rank holds the sum over ranks, bit-identical
            want = sum(dense_of(q).double() for q in range(world))
            assert torch.allclose(o["dense"].double().cpu(), want, rtol=1e-5, atol=1e-5)
            assert torch.equal(o["dense"], first[0]["dense"])
        # gate gradients are replicated: identical bits on every rank
        assert torch.equal(o["g_gate"], first[0]["g_gate"])
    assert not bad, bad


@pytest.mark.parametrize("world,precision,gate,ffn,rf,rb", [
    (2, "f32", "noisy_topk", "simple", 1, 1),
    (2, "bf16", "sigmoid_topk", "gated3", 2, 3),
    (4, "bf16", "noisy_topk", "simple", 3, 2),
    (4, "f32", "sigmoid_topk", "gated3", 2, 3),
    (8, "bf16", "expert_choice", "gated3", 2, 1),
    (8, "f32", "cosine_topk", "simple", 1, 2),
    (8, "bf16", "noisy_topk", "gated3", 1, 1),
])
def test_local_ep_matches_restatement(world, precision, gate, ffn, rf, rb):
    _run(world, precision, gate, ffn, rf, rb)


def test_local_ep_top1_unit_weight_path():
    """Switch top-1 (configs[1]'s gate): the I-order and its backward are row
    gathers / the dispatch kernel storing dO rows into the owners."""
    _run(4, "bf16", "noisy_topk", "simple", 1, 1, k=1)


def test_local_ep_dense_gradient_slices():
    """Dense-gradient allreduce slices in the backward's inter-link window
    (grad_partition.hpp) over the local group's collective."""
    _run(4, "bf16", "sigmoid_topk", "simple", 2, 2, dense=3 * 4099)


def test_local_ep_split_local_first():
    """FSMOE_EP_SPLIT: own experts' rows first, the peers' share on a second
    stream (moe_layer.cpp, the local-first split)."""
    _run(2, "bf16", "noisy_topk", "simple", 1, 1, split=1)


@pytest.mark.parametrize("world,precision,gate,ffn,rf,rb,k", [
    (2, "bf16", "noisy_topk", "simple", 3, 2, 2),
    (4, "f32", "sigmoid_topk", "gated3", 2, 3, 2),
    (8, "bf16", "noisy_topk", "simple", 4, 4, 1),
    (4, "bf16", "expert_choice", "gated3", 1, 2, 2),
])
def test_local_ep_copy_engine_chunked_pipeline(world, precision, gate, ffn, rf, rb, k):
    """FSMOE_EP_TRANSPORT=ce: the dispatch-side exchanges move per pipeline
    chunk on the copy engines (fsmoe_peer_copy_rows) with stream-memory-op
    flags (fsmoe_peer_flag_write), GEMM chunk i waiting only for chunk i."""
    _run(world, precision, gate, ffn, rf, rb, k=k, transport="ce")


@pytest.mark.parametrize("world,transport,rf,rb", [
    (8, "peer", 1, 1), (8, "peer", 2, 2), (8, "ce", 2, 2), (4, "ce", 3, 2)])
def test_local_ep_one_expert_per_rank(world, transport, rf, rb):
    """configs[2] on 8 GPUs holds one expert per rank (E_l = 1): top-2 noisy
    SwiGLU with both exchange transports and chunked pipelines."""
    _run(world, "bf16", "noisy_topk", "gated3", rf, rb, transport=transport, experts_per_rank=1)
