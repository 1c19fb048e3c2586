"""Time / profile the gate (K1) at the bench shape (T=16384, M=1024, E=16,
noisy top-1, bf16 tokens): pruned vs exhaustive exact paths."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10714_b200 import ops  # noqa: E402


def run(T=16384, M=1024, E=16, k=1, kind="noisy_topk", reps=5):
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    ws = ((torch.rand(M, E, device="cuda", generator=g, dtype=torch.float64) * 2 - 1) / M ** 0.5)
    wn = ((torch.rand(M, E, device="cuda", generator=g, dtype=torch.float64) * 2 - 1) / M ** 0.5)
    out = {}
    for path in ("pruned", "simt", "unfused", "exhaustive"):
        os.environ.pop("FSMOE_GATE_EXHAUSTIVE", None)
        os.environ.pop("FSMOE_GATE_UNFUSED", None)
        os.environ.pop("FSMOE_GATE_SIMT", None)
        if path == "simt":
            os.environ["FSMOE_GATE_SIMT"] = "1"
        if path == "exhaustive":
            os.environ["FSMOE_GATE_EXHAUSTIVE"] = "1"
        if path == "unfused":
            os.environ["FSMOE_GATE_UNFUSED"] = "1"
        r = ops.gate(kind, k, 7, x, ws, wn, save=True)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            r = ops.gate(kind, k, 7, x, ws, wn, save=True, check=False)
        e.record()
        torch.cuda.synchronize()
        out[path] = (s.elapsed_time(e) / reps * 1e3, r)
        print(f"{path}: {out[path][0]:.1f} us per gate call")
    a = out["pruned"][1]
    for other in ("simt", "unfused", "exhaustive"):
        b = out[other][1]
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
        print(f"pruned vs {other}: identical picks; max weight diff",
              (a[2] - b[2]).abs().max().item())
        for key in a[3]:
            print(f"  saved {key}: max diff", (a[3][key] - b[3][key]).abs().max().item())


if __name__ == "__main__":
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    print("configs[1] shape: T 16384, M 1024, E 16, top-1")
    run(reps=reps)
    print("configs[2] shape: T 32768, M 4096, E 8, top-2")
    run(T=32768, M=4096, E=8, k=2, reps=reps)
