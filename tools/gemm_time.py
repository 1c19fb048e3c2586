"""Time each of the six expert-FFN GEMM launches of one bench step
(configs[1]: E=16, C=1024, M=1024, H=4096) with CUDA events, 20 reps each,
and print us + PFLOP/s per launch."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10714_b200 import ops  # noqa: E402


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


def main(ffn="simple"):
    E, C, M, H = 16, 1024, 1024, 4096
    if ffn == "mixtral":  # configs[2] per GPU at N=4: 2 local experts x 4 sources x C 8192
        ffn, E, C, M, H = "gated3", 2, 32768, 4096, 14336
    N1 = H if ffn == "simple" else 2 * H
    bf = torch.bfloat16
    X = torch.randn(E, C, M, device="cuda").to(bf)
    W1 = (torch.randn(E, N1, M, device="cuda") / 32).to(bf)
    W2 = (torch.randn(E, M, H, device="cuda") / 64).to(bf)
    Z = torch.empty(E, C, N1, device="cuda", dtype=bf)
    Hh = torch.empty(E, C, H, device="cuda", dtype=bf)
    O = torch.empty(E, C, M, device="cuda", dtype=bf)
    dO = torch.randn(E, C, M, device="cuda").to(bf)
    dX = torch.empty_like(O)
    gw1 = torch.empty(E, N1, M, device="cuda")
    gw2 = torch.empty(E, M, H, device="cuda")
    fwd1_epi = "gelu_fwd" if ffn == "simple" else "swiglu_fwd"
    bwd_epi = "gelu_bwd" if ffn == "simple" else "swiglu_bwd"
    reps = 20 if C * M * H <= 2 ** 32 else 5
    launches = {
        "fwd1": lambda: ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=N1, n_w=E,
                                         epi=fwd1_epi, D2=Hh, ldd2=H),
        "fwd1_plain": lambda: ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=N1, n_w=E),
        "fwd2": lambda: ops.grouped_gemm("row", Hh, W2, O, nblk=E, rows=C, K=H, N=M, n_w=E),
        "wgrad2": lambda: ops.grouped_gemm("k", dO, Hh, gw2, nblk=E, rows=C, Mo=M, No=H, n_w=E,
                                           epi="store_f32"),
        "dgrad2": lambda: ops.grouped_gemm("row", dO, W2, Z, nblk=E, rows=C, K=M, N=H, n_w=E,
                                           b_mn_major=True, epi=bwd_epi, Zin=Z, ldz=N1, ldd=N1),
        "wgrad1": lambda: ops.grouped_gemm("k", Z, X, gw1, nblk=E, rows=C, Mo=N1, No=M, n_w=E,
                                           epi="store_f32"),
        "dgrad1": lambda: ops.grouped_gemm("row", Z, W1, dX, nblk=E, rows=C, K=N1, N=M, n_w=E,
                                           b_mn_major=True),
    }
    flops = 2.0 * E * C * M * H
    # (gated3: fwd1 / dgrad2 / wgrad1 do twice this; printed rates use 2*E*C*M*H)
    tot = 0.0
    for name, fn in launches.items():
        us = t(fn, reps)
        if name != "fwd1_plain":
            tot += us
        print(f"{name:11s} {us:8.1f} us  {flops / (us * 1e-6) / 1e15:.3f} PFLOP/s")
    print(f"six launches {tot:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "simple")
