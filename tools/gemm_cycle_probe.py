"""The six configs[2] expert GEMMs timed two ways in one process, each for a
few seconds of steady power-capped running: (a) every launch repeated back
to back (bench.py's roofline leg), (b) the six cycled in step order (what the
step does). Prints ms per six-launch set and the median SM clock of each."""
import os
import statistics
import subprocess
import sys
import tempfile
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10714_b200 import ops  # noqa: E402

E, C, M, H = 8, 8192, 4096, 14336
N1 = 2 * H


def clocks(fn, seconds):
    fd, path = tempfile.mkstemp()
    os.close(fd)
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "100", "-i", "0"], stdout=open(path, "w"))
    try:
        out = fn(seconds)
    finally:
        p.terminate()
        p.wait()
    vals = []
    for ln in open(path):
        try:
            vals.append(tuple(float(v) for v in ln.split(",")))
        except ValueError:
            pass
    os.unlink(path)
    vals = vals[3:] or vals
    return out, statistics.median(v[0] for v in vals), statistics.median(v[1] for v in vals)


def main():
    seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
    bf = torch.bfloat16
    torch.manual_seed(0)
    X = torch.randn(E, C, M, device="cuda").to(bf)
    W1 = (torch.randn(E, N1, M, device="cuda") / 64).to(bf)
    W2 = (torch.randn(E, M, H, device="cuda") / 128).to(bf)
    Z = torch.empty(E, C, N1, device="cuda", dtype=bf)
    Hh = torch.empty(E, C, H, device="cuda", dtype=bf)
    O = torch.empty(E, C, M, device="cuda", dtype=bf)
    dO = torch.randn(E, C, M, device="cuda").to(bf)
    dZ = torch.empty_like(Z)
    dX = torch.empty_like(O)
    gw1 = torch.empty(E, N1, M, device="cuda")
    gw2 = torch.empty(E, M, H, device="cuda")
    L = [
        lambda: ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=N1, n_w=E, epi="swiglu_fwd", D2=Hh, ldd2=H),
        lambda: ops.grouped_gemm("row", Hh, W2, O, nblk=E, rows=C, K=H, N=M, n_w=E),
        lambda: ops.grouped_gemm("k", dO, Hh, gw2, nblk=E, rows=C, Mo=M, No=H, n_w=E, epi="store_f32"),
        lambda: ops.grouped_gemm("row", dO, W2, dZ, nblk=E, rows=C, K=M, N=H, n_w=E, b_mn_major=True,
                                 epi="swiglu_bwd", Zin=Z, ldz=N1, ldd=N1),
        lambda: ops.grouped_gemm("k", dZ, X, gw1, nblk=E, rows=C, Mo=N1, No=M, n_w=E, epi="store_f32"),
        lambda: ops.grouped_gemm("row", dZ, W1, dX, nblk=E, rows=C, K=N1, N=M, n_w=E, b_mn_major=True),
    ]

    def timed(order):
        def run(seconds):
            for f in order[:6]:
                f()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 0
            s.record()
            t_end = time.time() + seconds
            while time.time() < t_end:
                for f in order:
                    f()
                n += 1
                torch.cuda.synchronize()
            e.record()
            torch.cuda.synchronize()
            return s.elapsed_time(e) / n * 6 / len(order)
        return run

    reps = [f for f in L for _ in range(5)]
    for name, order in (("warm", L), ("cycled", L), ("5x each", reps), ("cycled", L), ("5x each", reps)):
        ms, clk, pw = clocks(timed(order), seconds)
        print(f"{name:8s}: {ms:8.2f} ms per six-launch set, SM {clk:.0f} MHz, {pw:.0f} W", flush=True)


if __name__ == "__main__":
    main()
