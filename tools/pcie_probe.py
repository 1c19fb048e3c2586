"""Host<->device copy bandwidth for the e2e path (pinned buffers, 32 MB
bf16 copies like x / dy / dx of the bench step)."""
import torch


def bw(fn, nbytes, reps=20):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    return nbytes / (ms * 1e-3) / 1e9, ms


def main():
    n = 16384 * 1024
    h = [torch.empty(n, dtype=torch.bfloat16).pin_memory() for _ in range(3)]
    d = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    print("H2D 1x32MB      %.1f GB/s (%.3f ms)" % bw(lambda: d[0].copy_(h[0], non_blocking=True), 2 * n))
    print("D2H 1x32MB      %.1f GB/s (%.3f ms)" % bw(lambda: h[0].copy_(d[0], non_blocking=True), 2 * n))

    def two():
        with torch.cuda.stream(s1):
            d[0].copy_(h[0], non_blocking=True)
        with torch.cuda.stream(s2):
            d[1].copy_(h[1], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    print("H2D 2x32MB on 2 streams %.1f GB/s (%.3f ms)" % bw(two, 4 * n))

    def both():
        with torch.cuda.stream(s1):
            d[0].copy_(h[0], non_blocking=True)
            d[1].copy_(h[1], non_blocking=True)
        with torch.cuda.stream(s2):
            h[2].copy_(d[2], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    print("H2D 64MB + D2H 32MB concurrently: %.1f GB/s total (%.3f ms)" % bw(both, 6 * n))


if __name__ == "__main__":
    main()
