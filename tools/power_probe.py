"""Sustained throughput, SM clock and board power of the Mixtral-shape
(configs[2], N = 1: 8 experts x C 8192 rows) expert GEMMs: ours
(grouped_gemm_kernel, every launch of the step) against cuBLAS (torch.bmm,
plain bf16 stores) on the same shapes, each run back to back for a few
seconds while nvidia-smi samples clocks and power. Under the power cap the
step's speed is set by energy per flop, so this separates "fewer joules
per flop" work (DRAM over-read, epilogue) from mainloop work.

    python tools/power_probe.py [seconds] [variants...]
variants: ours, cublas, ours_bn256, ours_bn512, ours_dbg4 (no output stores)
"""
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_10714_b200 import ops  # noqa: E402

E, C, M, H = 8, 8192, 4096, 14336
N1 = 2 * H
bf = torch.bfloat16


class Smi:
    def __enter__(self):
        fd, self.path = tempfile.mkstemp()
        os.close(fd)
        self.p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                                   "-lms", "50", "-i", "0"], stdout=open(self.path, "w"))
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.p.terminate()
        self.p.wait()
        rows = []
        for ln in open(self.path):
            try:
                c, p = (float(v) for v in ln.split(","))
                rows.append((c, p))
            except ValueError:
                pass
        os.unlink(self.path)
        self.rows = rows[6:] if len(rows) > 10 else rows


def run(fn, flops, seconds):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t_end = time.time() + 1.0
    while time.time() < t_end:  # warm to steady clocks
        fn()
        torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    with Smi() as smi:
        s.record()
        t_end = time.time() + seconds
        while time.time() < t_end:
            fn()
            n += 1
            if n % 4 == 0:
                torch.cuda.synchronize()
        e.record()
        torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    clk = statistics.median(r[0] for r in smi.rows) if smi.rows else None
    pw = statistics.median(r[1] for r in smi.rows) if smi.rows else None
    return {"ms": round(ms, 3), "tflops": round(flops / ms / 1e9, 1), "sm_mhz": clk, "power_w": pw,
            "tflops_per_ghz": round(flops / ms / 1e9 / (clk / 1000.0), 1) if clk else None}


def main():
    seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
    variants = sys.argv[2:] or ["ours", "cublas"]
    torch.manual_seed(0)
    X = (torch.randn(E, C, M, device="cuda")).to(bf)
    W1 = (torch.randn(E, N1, M, device="cuda") / 64).to(bf)
    W2 = (torch.randn(E, M, H, device="cuda") / 128).to(bf)
    Z = torch.empty(E, C, N1, device="cuda", dtype=bf)
    Hh = torch.randn(E, C, H, device="cuda").to(bf)
    O = torch.empty(E, C, M, device="cuda", dtype=bf)
    dO = torch.randn(E, C, M, device="cuda").to(bf)
    dX = torch.empty_like(O)
    gw1 = torch.empty(E, N1, M, device="cuda")
    gw2 = torch.empty(E, M, H, device="cuda")
    fl_1 = 2 * E * C * M * N1
    fl_2 = 2 * E * C * M * H
    out = {}

    def ours(force=None, dbg=0):
        kw = dict(force=force, dbg=dbg)
        ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=N1, n_w=E, epi="swiglu_fwd", D2=Hh,
                         ldd2=H, **kw)
        Zc = Z
        return [
            ("fwd1", fl_1, lambda: ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=N1, n_w=E,
                                                    epi="swiglu_fwd", D2=Hh, ldd2=H, **kw)),
            ("fwd2", fl_2, lambda: ops.grouped_gemm("row", Hh, W2, O, nblk=E, rows=C, K=H, N=M, n_w=E, **kw)),
            ("wgrad2", fl_2, lambda: ops.grouped_gemm("k", dO, Hh, gw2, nblk=E, rows=C, Mo=M, No=H, n_w=E,
                                                      epi="store_f32", **kw)),
            ("dgrad2", fl_2, lambda: ops.grouped_gemm("row", dO, W2, Zc, nblk=E, rows=C, K=M, N=H, n_w=E,
                                                      b_mn_major=True, epi="swiglu_bwd", Zin=Z, ldz=N1,
                                                      ldd=N1, **kw)),
            ("wgrad1", fl_1, lambda: ops.grouped_gemm("k", Zc, X, gw1, nblk=E, rows=C, Mo=N1, No=M, n_w=E,
                                                      epi="store_f32", **kw)),
            ("dgrad1", fl_1, lambda: ops.grouped_gemm("row", Zc, W1, dX, nblk=E, rows=C, K=N1, N=M, n_w=E,
                                                      b_mn_major=True, **kw)),
        ]

    for v in variants:
        if v == "cublas":
            calls = [
                ("fwd1", fl_1, lambda: torch.bmm(X, W1.transpose(1, 2), out=Z)),
                ("fwd2", fl_2, lambda: torch.bmm(Hh, W2.transpose(1, 2), out=O)),
                ("wgrad2", fl_2, lambda: torch.bmm(dO.transpose(1, 2), Hh)),
                ("dgrad2", fl_2, lambda: torch.bmm(dO, W2)),
                ("wgrad1", fl_1, lambda: torch.bmm(Z.transpose(1, 2), X)),
                ("dgrad1", fl_1, lambda: torch.bmm(Z, W1, out=dX)),
            ]
        elif v == "ours":
            calls = ours()
        elif v == "ours_bn256":
            calls = ours(force=(2, 256))
        elif v == "ours_bn512":
            calls = ours(force=(2, 512))
        elif v == "ours_dbg4":
            calls = ours(dbg=4)
        else:
            raise SystemExit(f"unknown variant {v}")
        res = {}
        for name, fl, fn in calls:
            res[name] = run(fn, fl, seconds)
            print(v, name, res[name], flush=True)
        out[v] = res
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "power_probe.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
