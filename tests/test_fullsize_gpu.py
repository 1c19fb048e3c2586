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
