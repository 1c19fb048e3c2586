"""TEST INFRASTRUCTURE ONLY — the body of __graft_entry__.smoke().

One small MoE-layer forward + backward on cuda:0 through the product path
(libfsmoe.so C++ layer -> libfsmoe_cuda.so sm_100a kernels), routing checked
pick-by-pick against the CPU oracle (test infrastructure) and outputs /
gradients against the fp64 restatement."""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # repo root


def run() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("smoke() needs a CUDA device (there is no CPU fallback)")
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, ROOT)
    import layer_oracle  # test infrastructure (checker only)
    import pyoracle

    from paper_2501_10714_b200.layer import MoEConfig, MoELayer

    torch.cuda.set_device(0)
    T, M, H, E, k = 512, 256, 512, 8, 2
    cfg = MoEConfig(tokens=T, model_dim=M, ffn_dim=H, experts=E, top_k=k, gate="noisy_topk",
                    ffn="simple", precision="bf16", seed=7)
    layer = MoELayer(cfg, init_seed=3)
    g = torch.Generator().manual_seed(5)
    x = (torch.rand(T, M, generator=g) * 2 - 1).to("cuda", torch.bfloat16)
    dy = (torch.rand(T, M, generator=g) * 2 - 1).to("cuda", torch.bfloat16)
    y = layer.forward(x)
    dx = layer.backward(dy)
    torch.cuda.synchronize()

    W1 = layer.w1.double().cpu().numpy()
    W2 = layer.w2.double().cpu().numpy()
    yr, cache = layer_oracle.forward(x.double().cpu().numpy(), "noisy_topk", k, 7, layer.capacity,
                                     layer.w_gate.cpu().numpy(), layer.w_noise.cpu().numpy(),
                                     None, W1, W2, "simple", pyoracle.Oracle("port"))
    ref = layer_oracle.backward(cache, dy.double().cpu().numpy(), "noisy_topk", k, layer.capacity,
                                layer.w_gate.cpu().numpy(), layer.w_noise.cpu().numpy(), None,
                                W1, W2, "simple")
    n = cache.picks.token.size
    tok = layer.buffer("pick_token", torch.int32)[:n].cpu().numpy()
    exp = layer.buffer("pick_expert", torch.int32)[:n].cpu().numpy()
    slot = layer.buffer("slot_of_pick", torch.int32)[:n].cpu().numpy()
    assert np.array_equal(tok, cache.picks.token), "routing tokens differ from the oracle"
    assert np.array_equal(exp, cache.picks.expert), "routing experts differ from the oracle"
    assert np.array_equal(slot, cache.disp.slot_of_pick), "capacity slots differ from the oracle"

    def rel(a, b):
        a = a.double().cpu().numpy()
        return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))

    errs = {"y": rel(y, yr), "dx": rel(dx, ref["dx"]), "g_w1": rel(layer.g_w1, ref["g_w1"]),
            "g_w2": rel(layer.g_w2, ref["g_w2"]), "g_gate": rel(layer.g_gate, ref["g_gate"])}
    bad = {k_: v for k_, v in errs.items() if not v < 3e-2}
    layer.close()
    if bad:
        raise AssertionError(f"smoke parity failed: {bad}")
    print(f"smoke ok: routing bit-exact ({n} picks), rel errs {errs}")


if __name__ == "__main__":
    run()
