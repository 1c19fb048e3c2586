"""Where the e2e gap of the configs[2] N = 1 step goes: the same layer timed
(A) on device-resident buffers, (B) through bench.py's e2e loop (pinned host
x / dy in, y / dx out, copy streams, triple-buffered), (C) the e2e loop's
stream / event structure with the copies left out. Alternating rounds,
~2 s of steps each, median SM clock per phase."""
import os
import statistics
import subprocess
import sys
import tempfile
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def clocked(fn):
    fd, path = tempfile.mkstemp()
    os.close(fd)
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "100", "-i", "0"], stdout=open(path, "w"))
    try:
        ms = fn()
    finally:
        p.terminate()
        p.wait()
    v = []
    for ln in open(path):
        try:
            v.append(tuple(float(a) for a in ln.split(",")))
        except ValueError:
            pass
    os.unlink(path)
    v = v[3:] or v
    return ms, statistics.median(a[0] for a in v), statistics.median(a[1] for a in v)


def main():
    W = bench.WORKLOADS["mixtral"]
    T, M = W["tokens_per_gpu"], W["d_model"]
    from paper_2501_10714_b200.layer import MoELayer
    layer = MoELayer(bench.layer_config(W, None, 1, 1, ""), None, init_seed=1)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    NB = 3
    xh = x.cpu().pin_memory()
    dyh = dy.cpu().pin_memory()
    xd = [torch.empty_like(x) for _ in range(NB)]
    dyd = [torch.empty_like(x) for _ in range(NB)]
    yd = [torch.empty_like(x) for _ in range(NB)]
    dxd = [torch.empty_like(x) for _ in range(NB)]
    yh = [torch.empty(x.shape, dtype=x.dtype).pin_memory() for _ in range(NB)]
    dxh = [torch.empty(x.shape, dtype=x.dtype).pin_memory() for _ in range(NB)]
    comp = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    E = lambda: torch.cuda.Event()  # noqa: E731
    ev_x, ev_dy, ev_y, ev_done, ev_free = ([E() for _ in range(NB)] for _ in range(5))
    for e in ev_free:
        e.record(s_out)

    def plain(n):
        for _ in range(n):
            layer.forward(x, y)
            layer.backward(dy, dx)

    def e2e(n, copies):
        for i in range(n):
            b = i % NB
            with torch.cuda.stream(s_in):
                s_in.wait_event(ev_free[b])
                if copies:
                    xd[b].copy_(xh, non_blocking=True)
                ev_x[b].record(s_in)
                if copies:
                    dyd[b].copy_(dyh, non_blocking=True)
                ev_dy[b].record(s_in)
            comp.wait_event(ev_x[b])
            layer.forward(xd[b] if copies else x, yd[b])
            ev_y[b].record(comp)
            comp.wait_event(ev_dy[b])
            layer.backward(dyd[b] if copies else dy, dxd[b])
            ev_done[b].record(comp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_y[b])
                if copies:
                    yh[b].copy_(yd[b], non_blocking=True)
                s_out.wait_event(ev_done[b])
                if copies:
                    dxh[b].copy_(dxd[b], non_blocking=True)
                ev_free[b].record(s_out)
        comp.wait_stream(s_out)

    def timed(fn, n=40):
        def go():
            fn(4)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn(n)
            e.record()
            torch.cuda.synchronize()
            return s.elapsed_time(e) / n
        return go

    t_end = time.time() + 3
    while time.time() < t_end:
        plain(2)
        torch.cuda.synchronize()
    for rnd in range(3):
        for name, fn in (("A device", plain), ("B e2e", lambda n: e2e(n, True)),
                         ("C e2e-structure", lambda n: e2e(n, False))):
            ms, clk, pw = clocked(timed(fn))
            print(f"round {rnd} {name:16s} {ms:7.2f} ms/step  SM {clk:.0f} MHz  {pw:.0f} W", flush=True)


if __name__ == "__main__":
    main()
