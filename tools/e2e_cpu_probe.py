"""Is the e2e loop CPU-launch-bound? Time host-side enqueue of the bench's
double-buffered e2e step against its device time."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10714_b200.layer import MoEConfig, MoELayer  # noqa: E402


def main():
    cfg = MoEConfig(tokens=16384, model_dim=1024, ffn_dim=4096, experts=16, top_k=1)
    layer = MoELayer(cfg, init_seed=1)
    x = torch.randn(16384, 1024, device="cuda").to(torch.bfloat16)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    for _ in range(3):
        layer.forward(x, y)
        layer.backward(x, dx)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 50
    for _ in range(n):
        layer.forward(x, y)
        layer.backward(x, dx)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"enqueue {1e3 * (t1 - t0) / n:.3f} ms/step, wall {1e3 * (t2 - t0) / n:.3f} ms/step")


if __name__ == "__main__":
    main()
