"""Is the K=1024 expert GEMM epilogue-bound? Time the same grouped GEMM
(E=16 blocks of C=1024 rows, K=1024, N=4096) with each epilogue."""
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
    E, C, M, H = 16, 1024, 1024, 4096
    bf = torch.bfloat16
    X = torch.randn(E, C, M, device="cuda").to(bf)
    W1 = (torch.randn(E, H, M, device="cuda") / 32).to(bf)
    W2 = (torch.randn(E, M, H, device="cuda") / 64).to(bf)
    Z = torch.empty(E, C, H, device="cuda", dtype=bf)
    Hh = torch.empty(E, C, H, device="cuda", dtype=bf)
    dO = torch.randn(E, C, M, device="cuda").to(bf)
    Zf = torch.empty(E, C, H, device="cuda", dtype=torch.float32)
    gw2 = torch.empty(E, M, H, device="cuda")
    flops = 2 * E * C * M * H
    cases = {
        "fwd1 gelu_fwd": lambda: ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=H, n_w=E,
                                                  epi="gelu_fwd", D2=Hh, ldd2=H),
        "fwd1 store_bf16": lambda: ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=H, n_w=E),
        "fwd1 store_f32": lambda: ops.grouped_gemm("row", X, W1, Zf, nblk=E, rows=C, K=M, N=H, n_w=E,
                                                   epi="store_f32"),
        "dgrad2 gelu_bwd": lambda: ops.grouped_gemm("row", dO, W2, Z, nblk=E, rows=C, K=M, N=H, n_w=E,
                                                    b_mn_major=True, epi="gelu_bwd", Zin=Z, ldz=H),
        "dgrad2 store_bf16": lambda: ops.grouped_gemm("row", dO, W2, Z, nblk=E, rows=C, K=M, N=H, n_w=E,
                                                      b_mn_major=True),
        "wgrad2 f32": lambda: ops.grouped_gemm("k", dO, Hh, gw2, nblk=E, rows=C, Mo=M, No=H, n_w=E,
                                               epi="store_f32"),
    }
    for name, fn in cases.items():
        us = t(fn)
        print(f"{name:20s} {us:7.1f} us  {flops / us / 1e6:7.1f} TFLOP/s")


if __name__ == "__main__":
    main()
