"""Epilogue cost at the Mixtral shape: SwiGLU fwd / bwd epilogues vs a plain
bf16 store on the same grouped GEMMs (8 experts x 8192 rows, M 4096, H 14336)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10714_b200 import ops  # noqa: E402
from epi_probe import t  # noqa: E402


def main():
    E, C, M, H = 8, 8192, 4096, 14336
    bf = torch.bfloat16
    X = torch.randn(E, C, M, device="cuda").to(bf)
    W1 = (torch.randn(E, 2 * H, M, device="cuda") / 64).to(bf)
    W2 = (torch.randn(E, M, H, device="cuda") / 128).to(bf)
    Z = torch.empty(E, C, 2 * H, device="cuda", dtype=bf)
    Hh = torch.empty(E, C, H, device="cuda", dtype=bf)
    dO = torch.randn(E, C, M, device="cuda").to(bf)
    f1 = 2 * E * C * M * 2 * H
    f2 = 2 * E * C * M * H
    cases = [
        ("fwd1 swiglu_fwd", f1, lambda: ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=2 * H, n_w=E,
                                                         epi="swiglu_fwd", D2=Hh, ldd2=H)),
        ("fwd1 store_bf16", f1, lambda: ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=2 * H, n_w=E)),
        ("dgrad2 swiglu_bwd", f2, lambda: ops.grouped_gemm("row", dO, W2, Z, nblk=E, rows=C, K=M, N=H, n_w=E,
                                                           b_mn_major=True, epi="swiglu_bwd", Zin=Z,
                                                           ldz=2 * H, ldd=2 * H)),
        ("dgrad2 store_bf16", f2, lambda: ops.grouped_gemm("row", dO, W2, Hh, nblk=E, rows=C, K=M, N=H, n_w=E,
                                                           b_mn_major=True)),
    ]
    for name, fl, fn in cases:
        us = t(fn, reps=5)
        print(f"{name:20s} {us / 1e3:8.2f} ms  {fl / us / 1e6:7.1f} TFLOP/s")


if __name__ == "__main__":
    main()
