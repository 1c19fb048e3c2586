"""Gate backward on the tensor cores (bf16 tokens: x^T [G1 | G2] as a
k-grouped tcgen05 GEMM of a three-term bf16 split of G, dx += G W^T through
the AddBF16 epilogue) against the fp32 SIMT kernels on the same values
(x given as fp32, which takes the SIMT path). The parameter gradients agree
to fp32 accuracy; dx to its bf16 rounding."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = a.double(), b.double()
    return ((a - b).abs().max() / b.abs().max().clamp_min(1e-300)).item()


@pytest.mark.parametrize("kind,T,M,E,k", [("noisy_topk", 4096, 512, 8, 2), ("noisy_topk", 1000, 1600, 8, 2),
                                          ("sigmoid_topk", 2048, 1024, 16, 4), ("noisy_topk", 640, 256, 4, 2)])
def test_gate_bwd_tc_matches_simt(kind, T, M, E, k):
    from paper_2501_10714_b200 import ops
    g = np.random.default_rng(3)
    x = torch.randn(T, M, device="cuda").to(torch.bfloat16)
    ws = torch.from_numpy((g.random((M, E)) * 2 - 1) / np.sqrt(M)).cuda()
    wn = torch.from_numpy((g.random((M, E)) * 2 - 1) / np.sqrt(M)).cuda() if kind == "noisy_topk" else None
    tok, exp, w, saved = ops.gate(kind, k, 7, x, ws, wn, save=True)
    dw = torch.from_numpy(g.standard_normal(w.shape)).cuda()
    dx0 = torch.randn(T, M, device="cuda").to(torch.bfloat16)
    out = {}
    for name, xx, dx in (("tc", x, dx0.clone()), ("simt", x.float(), dx0.float())):
        gws = torch.zeros_like(ws)
        gwn = torch.zeros_like(wn) if wn is not None else None
        ops.gate_bwd(kind, k, 7, xx, ws, wn, None, tok, exp, w, dw, saved, dx, gws, gwn)
        torch.cuda.synchronize()
        out[name] = (gws, gwn, dx)
    assert _rel(out["tc"][0], out["simt"][0]) < 1e-5
    if wn is not None:
        assert _rel(out["tc"][1], out["simt"][1]) < 1e-5
    # dx: the bf16 rounding of the fp32 SIMT result (one ulp, 2^-8 relative)
    ref = out["simt"][2]
    err = (out["tc"][2].double() - ref.double()).abs()
    assert bool((err <= ref.double().abs() * 2.0 ** -8 + 1e-6 * ref.double().abs().max()).all())
