import torch
E, C, M, H = 16, 1024, 1024, 4096
bf = torch.bfloat16
X = torch.randn(E, C, M, device="cuda").to(bf)
W1 = (torch.randn(E, H, M, device="cuda") / 32).to(bf)
Hh = torch.randn(E, C, H, device="cuda").to(bf)
W2 = (torch.randn(E, M, H, device="cuda") / 64).to(bf)
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3
fl = 2 * E * C * M * H
for name, fn in [("bmm X.W1^T (fwd1 shape)", lambda: torch.bmm(X, W1.transpose(1, 2))),
                 ("bmm H.W2^T (fwd2 shape)", lambda: torch.bmm(Hh, W2.transpose(1, 2))),
                 ("mm 16384x1024 . 1024x4096", lambda: X.view(-1, M) @ W1[0].T.contiguous()),
                 ("mm 8192^2 x 8192", lambda: torch.mm(torch.empty(8192, 8192, device='cuda', dtype=bf), torch.empty(8192, 8192, device='cuda', dtype=bf)))]:
    us = t(fn)
    f = fl if "8192" not in name else 2 * 8192 ** 3
    print(f"{name:32s} {us:8.1f} us {f / us / 1e6:7.1f} TFLOP/s")
