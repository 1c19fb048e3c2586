"""L2 eviction-hint probe for the configs[2] (N = 1) expert GEMMs: every
launch of the step under a set of measurement flags (fsmoe_gemm_desc::dbg
bits 16 = output stores evict_first, 32 = A loads evict_last, 64 = B loads
evict_last, 128 = B loads evict_first), one launch each, meant to run under

    ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --csv \
        --log-file gpurun_out/l2hint.csv python tools/l2hint_probe.py

and summarised with `python tools/l2hint_probe.py --summarise gpurun_out/l2hint.csv`.
The hint flags were removed from the kernel after this experiment (no
measurable gain, profiles/r02_gemm_experiments.md); the probe is kept as the
record of how it was measured.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

E, C, M, H = 8, 8192, 4096, 14336
N1 = 2 * H
ORDERS = [0, 16, 16 | 32, 16 | 64, 16 | 128, 32, 64, 16 | 32 | 128]
# algorithmic operand bytes per launch (A + B reads, bf16)
ALGO = {"fwd1": (E * C * M + E * N1 * M) * 2, "fwd2": (E * C * H + E * M * H) * 2,
        "wgrad2": (E * C * M + E * C * H) * 2, "dgrad2": (E * C * M + E * M * H + E * C * N1) * 2,
        "wgrad1": (E * C * N1 + E * C * M) * 2, "dgrad1": (E * C * N1 + E * N1 * M) * 2}
NAMES = ["fwd1", "fwd2", "wgrad2", "dgrad2", "wgrad1", "dgrad1"]


def run():
    import torch
    from paper_2501_10714_b200 import ops
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
    ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=N1, n_w=E, epi="swiglu_fwd", D2=Hh, ldd2=H)
    calls = {
        "fwd1": lambda o: ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=N1, n_w=E,
                                           epi="swiglu_fwd", D2=Hh, ldd2=H, dbg=o),
        "fwd2": lambda o: ops.grouped_gemm("row", Hh, W2, O, nblk=E, rows=C, K=H, N=M, n_w=E, dbg=o),
        "wgrad2": lambda o: ops.grouped_gemm("k", dO, Hh, gw2, nblk=E, rows=C, Mo=M, No=H, n_w=E,
                                             epi="store_f32", dbg=o),
        "dgrad2": lambda o: ops.grouped_gemm("row", dO, W2, dZ, nblk=E, rows=C, K=M, N=H, n_w=E,
                                             b_mn_major=True, epi="swiglu_bwd", Zin=Z, ldz=N1, ldd=N1,
                                             dbg=o),
        "wgrad1": lambda o: ops.grouped_gemm("k", Z, X, gw1, nblk=E, rows=C, Mo=N1, No=M, n_w=E,
                                             epi="store_f32", dbg=o),
        "dgrad1": lambda o: ops.grouped_gemm("row", Z, W1, dX, nblk=E, rows=C, K=N1, N=M, n_w=E,
                                             b_mn_major=True, dbg=o),
    }
    torch.cuda.synchronize()
    for name in NAMES:
        for o in ORDERS:
            calls[name](o)
    torch.cuda.synchronize()


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    ui = h.index("Metric Unit")
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
             "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    per = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi or "grouped_gemm" not in r[ki]:
            continue
        # bytes in bytes, durations in ms
        per.setdefault(int(r[ii]), {})[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    ids = sorted(per)[1:]  # the first launch initialises Z
    out = {}
    lines = ["| launch | dbg flags | ms (ncu) | DRAM read GB | x algorithmic |", "|---|---|---|---|---|"]
    k = 0
    for name in NAMES:
        for o in ORDERS:
            m = per[ids[k]]
            k += 1
            gb = m.get("dram__bytes_read.sum", 0.0) / 1e9
            t_ms = m.get("gpu__time_duration.sum", 0.0)
            ratio = gb * 1e9 / ALGO[name]
            out.setdefault(name, {})[str(o)] = {"ms": t_ms, "dram_read_gb": gb, "x_algorithmic": ratio}
            lines.append(f"| {name} | {o} | {t_ms:.3f} | {gb:.2f} | {ratio:.2f} |")
    print("\n".join(lines))
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--summarise":
        res = summarise(sys.argv[2])
        with open(os.path.splitext(sys.argv[2])[0] + ".json", "w") as f:
            json.dump(res, f, indent=1)
    else:
        run()
