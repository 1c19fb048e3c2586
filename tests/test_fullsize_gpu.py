"""Parity at BASELINE's full per-GPU sizes (the bench workloads), not just the
small shapes the fp64 restatement handles:

* routing for configs[1] (T 16384, M 1024, E 16, top-1 noisy, bf16 tokens) and
  the per-GPU routing of configs[2] (T 32768, M 4096, E 8, top-2 noisy):
  picks, weights and capacity slots against the C restatement of the
  reference (oracle/fsmoe_oracle.c, itself pinned to the reference's golden
  vectors) — bit-exact indices, weights within 1e-12;
* the whole configs[1] layer step (forward + backward through libfsmoe.so)
  against a torch fp32 composition of the same math on the GPU (TF32 off)
  with the executor's bf16 rounding points (Z, H, gelu', O, dO, dZ, dX):
  max |gpu - ref| / max |ref| < 1e-2 per tensor.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float((a.double() - b.double()).abs().max() / b.double().abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("T,M,E,k", [(16384, 1024, 16, 1), (32768, 4096, 8, 2)])
def test_routing_full_size_vs_port(T, M, E, k):
    import pyoracle
    from paper_2501_10714_b200 import ops
    g = np.random.default_rng(T + M + E + k)
    x = torch.from_numpy(g.standard_normal((T, M))).to(torch.bfloat16)
    ws = (g.random((M, E)) * 2 - 1) / np.sqrt(M)
    wn = (g.random((M, E)) * 2 - 1) / np.sqrt(M)
    orc = pyoracle.Oracle("port")
    o = orc.run_gate("noisy_topk", k, 7, x.double().numpy(), ws, wn, None)
    tok, exp, w = ops.gate("noisy_topk", k, 7, x.cuda(), torch.from_numpy(ws).cuda(),
                           torch.from_numpy(wn).cuda())
    np.testing.assert_array_equal(tok.cpu().numpy(), o.token)
    np.testing.assert_array_equal(exp.cpu().numpy(), o.expert)
    assert np.max(np.abs(w.cpu().numpy() - o.weight) / np.abs(o.weight)) <= 1e-12
    cap = -(-k * T // E)  # capacity_tokens at f = 1.0 (workload.cpp:43-51)
    slot, fill, dropped, _ = ops.assign(tok, exp, T, E, cap)
    # the reference's sequential fill: a pick is kept iff fewer than cap
    # earlier picks (in pick order) chose its expert
    e_np = o.expert.astype(np.int64)
    order = np.zeros_like(e_np)
    seen = np.zeros(E, dtype=np.int64)
    for i, e in enumerate(e_np):
        order[i] = seen[e]
        seen[e] += 1
    ref_slot = np.where(order < cap, e_np * cap + order, -1)
    np.testing.assert_array_equal(slot.cpu().numpy(), ref_slot)
    np.testing.assert_array_equal(fill.cpu().numpy(), np.minimum(seen, cap))
    assert int(dropped.item()) == int(np.sum(order >= cap))


def test_layer_step_config1_vs_torch_fp32():
    import pyoracle
    import torch.nn.functional as F
    from paper_2501_10714_b200.layer import MoEConfig, MoELayer
    torch.backends.cuda.matmul.allow_tf32 = False
    T, M, H, E = 16384, 1024, 4096, 16
    cfg = MoEConfig(tokens=T, model_dim=M, ffn_dim=H, experts=E, top_k=1, gate="noisy_topk",
                    ffn="simple", precision="bf16", seed=11)
    layer = MoELayer(cfg, init_seed=5)
    C = layer.capacity
    g = torch.Generator(device="cuda").manual_seed(21)
    x = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    y = layer.forward(x)
    dx = layer.backward(dy)
    torch.cuda.synchronize()

    # routing inside the layer == the C restatement, full size
    o = pyoracle.Oracle("port").run_gate("noisy_topk", 1, 11, x.double().cpu().numpy(),
                                         layer.w_gate.cpu().numpy(), layer.w_noise.cpu().numpy(), None)
    n = T
    tok = layer.buffer("pick_token", torch.int32)[:n]
    exp = layer.buffer("pick_expert", torch.int32)[:n]
    slot = layer.buffer("slot_of_pick", torch.int32)[:n]
    np.testing.assert_array_equal(tok.cpu().numpy(), o.token)
    np.testing.assert_array_equal(exp.cpu().numpy(), o.expert)
    assert np.all(o.weight == 1.0)  # top-1 masked softmax over one survivor

    # torch fp32 composition with the executor's bf16 rounding points
    keep = slot >= 0
    ts, ss = tok[keep].long(), slot[keep].long()
    X = torch.zeros(E * C, M, device="cuda")
    X[ss] = x[ts].float()
    Xe = X.view(E, C, M)
    W1, W2 = layer.w1.float(), layer.w2.float()            # [E, H, M], [E, M, H]
    Zb = torch.bmm(Xe, W1.transpose(1, 2)).bfloat16().float()
    Hb = F.gelu(Zb).bfloat16().float()
    Ob = torch.bmm(Hb, W2.transpose(1, 2)).bfloat16().float()
    y_ref = torch.zeros(T, M, device="cuda")
    y_ref[ts] = Ob.view(E * C, M)[ss]
    dO = torch.zeros(E * C, M, device="cuda")
    dO[ss] = dy[ts].float()
    dOe = dO.view(E, C, M)
    dH = torch.bmm(dOe, W2)
    pdf = torch.exp(-0.5 * Zb * Zb) * 0.3989422804014327
    gp = (0.5 * (1.0 + torch.erf(Zb * 0.7071067811865476)) + Zb * pdf).bfloat16().float()
    dZ = (dH * gp).bfloat16().float()
    dX = torch.bmm(dZ, W1).bfloat16().float()
    dx_ref = torch.zeros(T, M, device="cuda")
    dx_ref[ts] = dX.view(E * C, M)[ss]
    gw1 = torch.bmm(dZ.transpose(1, 2), Xe)
    gw2 = torch.bmm(dOe.transpose(1, 2), Hb)

    assert _rel(y.float(), y_ref) < 1e-2
    assert _rel(dx.float(), dx_ref) < 1e-2
    assert _rel(layer.g_w1, gw1) < 1e-2
    assert _rel(layer.g_w2, gw2) < 1e-2
    # dropped tokens produce zero output and zero input gradient
    dropped = ts.new_ones(T, dtype=torch.bool)
    dropped[ts] = False
    assert int(dropped.sum()) == T - int(keep.sum())
    assert float(y[dropped].abs().max() if dropped.any() else 0.0) == 0.0
    assert float(dx[dropped].abs().max() if dropped.any() else 0.0) == 0.0


def _silu(g):
    return g * torch.sigmoid(g)


@pytest.mark.parametrize("T,M,H,E,k,gate,ffn,proj_dim", [
    # configs[2]: the Mixtral-8x7B-shape layer, one GPU's share (32k tokens,
    # all 8 experts local = the per-GPU expert work of the 8-GPU job)
    (32768, 4096, 14336, 8, 2, "noisy_topk", "gated3", 0),
    # SURVEY C5 (configs[4]): every routing function at the GPT-2-XL shape
    (4096, 1600, 6400, 8, 2, "noisy_topk", "simple", 0),
    (4096, 1600, 6400, 8, 2, "sigmoid_topk", "simple", 0),
    (4096, 1600, 6400, 8, 2, "cosine_topk", "simple", 64),
    (4096, 1600, 6400, 8, 2, "expert_choice", "simple", 0),
])
def test_layer_step_full_size_weighted_vs_torch(T, M, H, E, k, gate, ffn, proj_dim):
    """The weighted top-k path at BASELINE's full sizes: routing against the C
    restatement (bit-exact picks, weights <= 1e-12), then forward + backward
    against a torch composition of the same math (expert GEMMs fp32, TF32
    off; gate fp64) with the executor's bf16 rounding points (Z, H, O, dO,
    dZ, dX): y, dx, expert-weight and gate-parameter gradients within 1e-2 of
    max |ref| (bf16 activations)."""
    import layer_oracle
    import pyoracle
    from paper_2501_10714_b200.layer import MoEConfig, MoELayer
    torch.backends.cuda.matmul.allow_tf32 = False
    cfg = MoEConfig(tokens=T, model_dim=M, ffn_dim=H, experts=E, top_k=k, gate=gate, ffn=ffn,
                    precision="bf16", seed=11, proj_dim=proj_dim)
    layer = MoELayer(cfg, init_seed=5)
    C = layer.capacity
    g = torch.Generator(device="cuda").manual_seed(31)
    x = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    y = layer.forward(x)
    dx = layer.backward(dy)
    torch.cuda.synchronize()

    ec = gate == "expert_choice"
    n = E * C if ec else T * k
    tok = layer.buffer("pick_token", torch.int32)[:n].long()
    exp = layer.buffer("pick_expert", torch.int32)[:n].long()
    w = layer.buffer("pick_weight", torch.float64)[:n]
    slot = layer.buffer("slot_of_pick", torch.int32)[:n].long()

    # routing == the C restatement of the reference (pinned to its goldens)
    wg = layer.w_gate.cpu().numpy()
    wn = layer.w_noise.cpu().numpy()
    pj = layer.proj.cpu().numpy() if layer.proj is not None else None
    xd = x.double()
    o = pyoracle.Oracle("port").run_gate(gate, C if ec else k, 11, xd.cpu().numpy(), wg,
                                         wn if gate == "noisy_topk" else None, pj)
    np.testing.assert_array_equal(tok.cpu().numpy(), o.token)
    np.testing.assert_array_equal(exp.cpu().numpy(), o.expert)
    assert np.max(np.abs(w.cpu().numpy() - o.weight) / np.abs(o.weight)) <= 1e-12

    # torch composition with the executor's bf16 rounding points
    keep = slot >= 0
    ts, ss, ws_ = tok[keep], slot[keep], w[keep]
    X = torch.zeros(E * C, M, device="cuda")
    X[ss] = x[ts].float()
    Xe = X.view(E, C, M)
    W1, W2 = layer.w1.float(), layer.w2.float()
    Zb = torch.bmm(Xe, W1.transpose(1, 2)).bfloat16().float()
    if ffn == "gated3":
        zz = Zb.view(E, C, H // 128, 2, 128)
        G, U = zz[:, :, :, 0, :].reshape(E, C, H), zz[:, :, :, 1, :].reshape(E, C, H)
        Hb = (_silu(G) * U).bfloat16().float()
    else:
        Hb = F.gelu(Zb).bfloat16().float()
    Ob = torch.bmm(Hb, W2.transpose(1, 2)).bfloat16().float()
    Of = Ob.view(E * C, M)
    y_ref = torch.zeros(T, M, device="cuda")
    y_ref.index_add_(0, ts, Of[ss] * ws_.float()[:, None])
    dyf = dy.float()
    dO = torch.zeros(E * C, M, device="cuda")
    dO[ss] = (dyf[ts] * ws_.float()[:, None]).bfloat16().float()
    dOe = dO.view(E, C, M)
    dH = torch.bmm(dOe, W2)
    if ffn == "gated3":
        sg = torch.sigmoid(G)
        dG = (dH * U * sg * (1.0 + G * (1.0 - sg))).bfloat16().float()
        dU = (dH * G * sg).bfloat16().float()
        dZ = torch.stack([dG.view(E, C, H // 128, 128), dU.view(E, C, H // 128, 128)], dim=3)
        dZ = dZ.reshape(E, C, 2 * H)
    else:
        pdf = torch.exp(-0.5 * Zb * Zb) * 0.3989422804014327
        gp = (0.5 * (1.0 + torch.erf(Zb * 0.7071067811865476)) + Zb * pdf).bfloat16().float()
        dZ = (dH * gp).bfloat16().float()
    dX = torch.bmm(dZ, W1).bfloat16().float()
    dx_ref = torch.zeros(T, M, device="cuda")
    dx_ref.index_add_(0, ts, dX.view(E * C, M)[ss])
    gw1 = torch.bmm(dZ.transpose(1, 2), Xe)
    gw2 = torch.bmm(dOe.transpose(1, 2), Hb)
    del Zb, Hb, dH, dZ, dX, X, Xe

    # gate backward in fp64, scores recomputed independently
    dw = torch.zeros(n, dtype=torch.float64, device="cuda")
    dw[keep] = (dyf[ts].double() * Of[ss].double()).sum(1)
    Wg, Wn = layer.w_gate, layer.w_noise
    dS = torch.zeros(T, E, dtype=torch.float64, device="cuda")
    if ec:
        wv, dv = w.view(E, C), dw.view(E, C)
        sig = (wv * dv).sum(1, keepdim=True)
        dS[tok.view(E, C), torch.arange(E, device="cuda")[:, None].expand(E, C)] = wv * (dv - sig)
    else:
        wv, dv, ev = w.view(T, k), dw.view(T, k), exp.view(T, k)
        if gate == "sigmoid_topk":
            vals = dv * wv * (1.0 - wv)
        else:
            vals = wv * (dv - (wv * dv).sum(1, keepdim=True))
        dS.scatter_(1, ev, vals)
    g_gate_ref = g_noise_ref = g_proj_ref = None
    if gate == "cosine_topk":
        P_ = layer.proj
        q = xd @ P_.T
        qn = q.norm(dim=1, keepdim=True)
        wnorm = Wg.norm(dim=0, keepdim=True)
        s = (q @ Wg) / (qn * wnorm)
        sdS = (dS * s).sum(1, keepdim=True)
        dq = (dS / (qn * wnorm)) @ Wg.T - sdS * q / qn ** 2
        g_gate_ref = (q / qn).T @ dS / wnorm - Wg * (dS * s).sum(0, keepdim=True) / wnorm ** 2
        g_proj_ref = dq.T @ xd
        dx_ref += (dq @ P_).float()
    else:
        g_gate_ref = xd.T @ dS
        dx_ref += (dS @ Wg.T).float()
        if gate == "noisy_topk":
            noise = torch.from_numpy(layer_oracle.noise_matrix(11, T, E)).cuda()
            spread = xd @ Wn
            dZn = dS * noise * torch.sigmoid(spread)
            g_noise_ref = xd.T @ dZn
            dx_ref += (dZn @ Wn.T).float()

    errs = {"y": _rel(y.float(), y_ref), "dx": _rel(dx.float(), dx_ref),
            "g_w1": _rel(layer.g_w1, gw1), "g_w2": _rel(layer.g_w2, gw2),
            "g_gate": _rel(layer.g_gate, g_gate_ref)}
    if g_noise_ref is not None:
        errs["g_noise"] = _rel(layer.g_noise, g_noise_ref)
    if g_proj_ref is not None:
        errs["g_proj"] = _rel(layer.g_proj, g_proj_ref)
    bad = {a: b for a, b in errs.items() if not b < 1e-2}
    assert not bad, errs
    # the gate really had a gradient (weighted top-k: not the k = 1 constant)
    assert float(layer.g_gate.abs().max()) > 0
    layer.close()
