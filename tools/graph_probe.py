"""How much of the N=1 step is launch / inter-kernel gap? Time forward +
backward eagerly and as a replayed CUDA graph (one rank: no peer-flag
epochs, so the step is capturable)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_10714_b200.layer import MoEConfig, MoELayer  # noqa: E402


def main():
    cfg = MoEConfig(tokens=16384, model_dim=1024, ffn_dim=4096, experts=16, top_k=1)
    layer = MoELayer(cfg, init_seed=1)
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(16384, 1024, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(16384, 1024, device="cuda", generator=g).to(torch.bfloat16)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            layer.forward(x, y)
            layer.backward(dy, dx)
    torch.cuda.synchronize()

    def timed(fn, n=50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    eager = timed(lambda: (layer.forward(x, y), layer.backward(dy, dx)))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        layer.forward(x, y)
        layer.backward(dy, dx)
    graph.replay()
    torch.cuda.synchronize()
    replay = timed(graph.replay)
    print(f"eager {eager:.3f} ms/step   graph replay {replay:.3f} ms/step")


if __name__ == "__main__":
    main()
