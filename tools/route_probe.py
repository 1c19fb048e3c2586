"""Time the permutation kernels at the bench shape (T=16384, M=1024, E=16,
C=1024, k=1, bf16) with CUDA events; HBM bytes per launch -> GB/s."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10714_b200 import ops  # noqa: E402


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


def main():
    T, M, E, k = 16384, 1024, 16, 1
    C = T * k // E
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    ws = (torch.rand(M, E, device="cuda", generator=g, dtype=torch.float64) * 2 - 1) / M ** 0.5
    wn = (torch.rand(M, E, device="cuda", generator=g, dtype=torch.float64) * 2 - 1) / M ** 0.5
    tok, exp, w = ops.gate("noisy_topk", k, 7, x, ws, wn)
    slot, fill, dropped, pos = ops.assign(tok, exp, T, E, C)
    tptr, tpick = ops.token_index(tok, T, token_major_k=k)
    buf = ops.dispatch(x, pos, tok, E, C)
    kept = int((slot >= 0).sum().item())
    b = 2
    res = {}
    res["assign"] = (t(lambda: ops.assign(tok, exp, T, E, C, check=False)), 0)
    res["dispatch"] = (t(lambda: ops.dispatch(x, pos, tok, E, C, out=buf)), (kept + E * C) * M * b)
    res["combine"] = (t(lambda: ops.combine(buf, tptr, tpick, slot, w, T, E, C)), (kept + T) * M * b)
    res["combine_bwd"] = (t(lambda: ops.combine_bwd(x, buf, pos, tok, w, E, C)), (2 * kept + E * C) * M * b)
    res["dispatch_bwd"] = (t(lambda: ops.dispatch_bwd(buf, tptr, tpick, slot, T, E, C)), (kept + T) * M * b)
    for name, (us, by) in res.items():
        print(f"{name:14s} {us:7.1f} us  {by / us / 1e3 if by else 0:7.0f} GB/s")


if __name__ == "__main__":
    main()
