"""Time the gate backward (fsmoe_gate_bwd) at the configs[2] per-GPU shape
(T 32768, M 4096, E 8, top-2 noisy, bf16 tokens); run under ncu for the
per-kernel split."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10714_b200 import ops  # noqa: E402


def main(T=32768, M=4096, E=8, k=2, reps=10):
    g = np.random.default_rng(1)
    x = torch.randn(T, M, device="cuda").to(torch.bfloat16)
    ws = torch.from_numpy((g.random((M, E)) * 2 - 1) / np.sqrt(M)).cuda()
    wn = torch.from_numpy((g.random((M, E)) * 2 - 1) / np.sqrt(M)).cuda()
    tok, exp, w, saved = ops.gate("noisy_topk", k, 7, x, ws, wn, save=True)
    dw = torch.randn_like(w)
    dx = torch.zeros_like(x)
    gws, gwn = torch.zeros_like(ws), torch.zeros_like(wn)
    fn = lambda: ops.gate_bwd("noisy_topk", k, 7, x, ws, wn, None, tok, exp, w, dw, saved, dx, gws, gwn)  # noqa: E731
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    print(f"gate_bwd T={T} M={M} E={E} k={k}: {s.elapsed_time(e) / reps * 1e3:.1f} us")
    s.record()
    for _ in range(reps):
        ops.gate("noisy_topk", k, 7, x, ws, wn, save=True)
    e.record()
    torch.cuda.synchronize()
    print(f"gate fwd (save): {s.elapsed_time(e) / reps * 1e3:.1f} us")


if __name__ == "__main__":
    main()
