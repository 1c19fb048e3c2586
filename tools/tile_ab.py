"""Same-process A/B of GEMM variants on the configs[1] (or --mixtral)
launches: each launch timed under the default heuristic and under forced
(ctas, bn) tiles or a measurement flag (dbg), interleaved rounds so clock
drift hits both alike.  --split: default vs two producer threads (dbg 8)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10714_b200 import ops  # noqa: E402


def t(fn, reps):
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
    mixtral = "--mixtral" in sys.argv
    E, C, M, H = (8, 8192, 4096, 14336) if mixtral else (16, 1024, 1024, 4096)
    ffn = "gated3" if mixtral else "simple"
    N1 = 2 * H if ffn == "gated3" else H
    bf = torch.bfloat16
    X = torch.randn(E, C, M, device="cuda").to(bf)
    W1 = ((torch.rand(E, N1, M, device="cuda") * 2 - 1) / M ** 0.5).to(bf)
    W2 = ((torch.rand(E, M, H, device="cuda") * 2 - 1) / H ** 0.5).to(bf)
    Z = torch.empty(E, C, N1, device="cuda", dtype=bf)
    Hh = torch.empty(E, C, H, device="cuda", dtype=bf)
    O = torch.empty(E, C, M, device="cuda", dtype=bf)
    dO = torch.randn(E, C, M, device="cuda").to(bf)
    dZ = torch.empty_like(Z)
    dX = torch.empty_like(O)
    gw1 = torch.empty(E, N1, M, device="cuda")
    gw2 = torch.empty(E, M, H, device="cuda")
    fe = "swiglu_fwd" if ffn == "gated3" else "gelu_fwd"
    be = "swiglu_bwd" if ffn == "gated3" else "gelu_bwd"
    ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=N1, n_w=E, epi=fe, D2=Hh, ldd2=H)
    split = "--split" in sys.argv

    def V(*force):
        if split:
            return [{}, {"dbg": 8}]
        return [{}] + ([{"force": force}] if force else [])

    L = {
        "fwd1": (lambda kw: ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=N1, n_w=E, epi=fe, D2=Hh,
                                            ldd2=H, **kw), V(2, 512)),
        "fwd2": (lambda kw: ops.grouped_gemm("row", Hh, W2, O, nblk=E, rows=C, K=H, N=M, n_w=E, **kw),
                 V(2, 256)),
        "wgrad2": (lambda kw: ops.grouped_gemm("k", dO, Hh, gw2, nblk=E, rows=C, Mo=M, No=H, n_w=E,
                                              epi="store_f32", **kw), V(2, 256)),
        "dgrad2": (lambda kw: ops.grouped_gemm("row", dO, W2, dZ, nblk=E, rows=C, K=M, N=H, n_w=E,
                                              b_mn_major=True, epi=be, Zin=Z, ldz=N1, ldd=N1, **kw),
                   V(2, 512) if ffn == "gated3" else V()),
        "wgrad1": (lambda kw: ops.grouped_gemm("k", Z, X, gw1, nblk=E, rows=C, Mo=N1, No=M, n_w=E,
                                              epi="store_f32", **kw), V(2, 256)),
        "dgrad1": (lambda kw: ops.grouped_gemm("row", Z, W1, dX, nblk=E, rows=C, K=N1, N=M, n_w=E,
                                              b_mn_major=True, **kw), V(2, 256)),
    }
    reps = 5 if mixtral else 40
    res = {}
    # (bitwise equality of the variants: tools/gemm_determinism.py)
    t_end = time.time() + 3.0
    while time.time() < t_end:  # steady clocks
        L["fwd2"][0]({})
        torch.cuda.synchronize()
    for rnd in range(6):
        for name, (fn, variants) in L.items():
            for v in variants:
                res.setdefault((name, str(v)), []).append(t(lambda: fn(v), reps))
    for (name, v), us in res.items():
        us = sorted(us)
        print(f"{name:7s} {v:20s} median {us[len(us) // 2]:9.1f} us  min {us[0]:9.1f}")


if __name__ == "__main__":
    main()
