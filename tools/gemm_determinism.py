"""Bitwise run-to-run determinism of the six expert-GEMM launches (configs[1]
or --mixtral shapes) under a given dbg flag: every launch run 3 times, each
output compared with the first run, and against the default (dbg 0) run."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10714_b200 import ops  # noqa: E402


def main():
    mixtral = "--mixtral" in sys.argv
    dbgs = [int(a) for a in sys.argv[1:] if a.isdigit()] or [0]
    E, C, M, H = (8, 8192, 4096, 14336) if mixtral else (16, 1024, 1024, 4096)
    ffn = "gated3" if mixtral else "simple"
    N1 = 2 * H if ffn == "gated3" else H
    bf = torch.bfloat16
    torch.manual_seed(0)
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
    L = {
        "fwd1": (lambda d: ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=N1, n_w=E, epi=fe, D2=Hh,
                                           ldd2=H, dbg=d), (Z, Hh)),
        "fwd2": (lambda d: ops.grouped_gemm("row", Hh, W2, O, nblk=E, rows=C, K=H, N=M, n_w=E, dbg=d), (O,)),
        "wgrad2": (lambda d: ops.grouped_gemm("k", dO, Hh, gw2, nblk=E, rows=C, Mo=M, No=H, n_w=E,
                                             epi="store_f32", dbg=d), (gw2,)),
        "dgrad2": (lambda d: ops.grouped_gemm("row", dO, W2, dZ, nblk=E, rows=C, K=M, N=H, n_w=E,
                                             b_mn_major=True, epi=be, Zin=Z, ldz=N1, ldd=N1, dbg=d), (dZ,)),
        "wgrad1": (lambda d: ops.grouped_gemm("k", Z, X, gw1, nblk=E, rows=C, Mo=N1, No=M, n_w=E,
                                             epi="store_f32", dbg=d), (gw1,)),
        "dgrad1": (lambda d: ops.grouped_gemm("row", Z, W1, dX, nblk=E, rows=C, K=N1, N=M, n_w=E,
                                             b_mn_major=True, dbg=d), (dX,)),
    }
    ok = True
    for name in ["fwd1", "fwd2", "wgrad2", "dgrad2", "wgrad1", "dgrad1"]:
        fn, outs = L[name]
        ref = None
        for d in [0] + dbgs:
            runs = []
            for _ in range(3):
                for o in outs:
                    o.fill_(float("nan")) if o.dtype != torch.float32 else o.fill_(float("nan"))
                fn(d)
                torch.cuda.synchronize()
                runs.append([o.clone() for o in outs])
            same = all(torch.equal(a, b) for r in runs[1:] for a, b in zip(runs[0], r))
            vs0 = ref is None or all(torch.equal(a, b) for a, b in zip(ref, runs[0]))
            ndiff = 0 if vs0 else sum(int((a != b).sum()) for a, b in zip(ref, runs[0]))
            if ref is None:
                ref = runs[0]
            print(f"{name:7s} dbg {d}: run-to-run identical {same}; equal to dbg 0 {vs0} ({ndiff} elements differ)",
                  flush=True)
            ok &= same and vs0
    print("ALL OK" if ok else "MISMATCH")


if __name__ == "__main__":
    main()
