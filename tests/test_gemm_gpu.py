"""Grouped expert GEMM (tcgen05 bf16 + fp32 SIMT check mode) vs a torch fp32
reference of the same op. The reference (FSMoE artifact) has no expert FFN
(it only counts GEMMs, proj/src/workload.cpp:70), so this is the
floating-point kernel's "plain PyTorch fp32 reference" check.

Tolerances: bf16 outputs rel 2e-2 of max|ref| (bf16 rounding of inputs and
outputs, fp32 accumulate); fp32 outputs of bf16 GEMMs rel 5e-3; fp32 check
mode rel 1e-5.
"""
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


def _ops():
    from paper_2501_10714_b200 import ops
    return ops


@pytest.fixture(params=["1x256", "2x256", "1x128", "2x128", "2x512"], autouse=True)
def gemm_ctas(request, monkeypatch):
    """Run every GEMM test on all tile variants: single-CTA (128 rows) and
    CTA-pair (256 rows, tcgen05 cta_group::2) x 256- and 128-column tiles,
    and the pair's 512-column tile (one accumulator, two MMAs per K step;
    every epilogue but GELU-backward, which keeps 256 columns)."""
    ctas, bn = request.param.split("x")
    from paper_2501_10714_b200 import ops
    monkeypatch.setattr(ops, "GEMM_FORCE", (int(ctas), int(bn)))
    return ctas


def _rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-30)).item()


def _rand(*shape, dtype=torch.bfloat16, scale=1.0):
    return (torch.randn(*shape, device="cuda") * scale).to(dtype)


@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("nblk,rows,K,N,n_w", [(3, 200, 192, 320, 3), (4, 256, 512, 512, 2),
                                               (2, 77, 64, 64, 1), (16, 128, 1024, 512, 16)])
def test_row_grouped_kmajor(precision, nblk, rows, K, N, n_w):
    ops = _ops()
    dt = torch.bfloat16 if precision == 0 else torch.float32
    torch.manual_seed(0)
    A = _rand(nblk, rows, K, dtype=dt)
    B = _rand(n_w, N, K, dtype=dt, scale=K ** -0.5)
    D = torch.empty(nblk, rows, N, device="cuda", dtype=dt)
    ops.grouped_gemm("row", A, B, D, nblk=nblk, rows=rows, K=K, N=N, n_w=n_w,
                     epi="store_bf16" if precision == 0 else "store_f32", precision=precision)
    torch.cuda.synchronize()
    ref = torch.stack([A[b].double() @ B[b % n_w].double().T for b in range(nblk)])
    assert _rel(D, ref) < (2e-2 if precision == 0 else 1e-5)


@pytest.mark.parametrize("precision", [0, 1])
def test_row_grouped_mnmajor_b(precision):
    ops = _ops()
    dt = torch.bfloat16 if precision == 0 else torch.float32
    nblk, rows, K, N, n_w = 4, 300, 256, 384, 2
    A = _rand(nblk, rows, K, dtype=dt)
    B = _rand(n_w, K, N, dtype=dt, scale=K ** -0.5)  # stored [w][K][N]
    D = torch.empty(nblk, rows, N, device="cuda", dtype=dt)
    ops.grouped_gemm("row", A, B, D, nblk=nblk, rows=rows, K=K, N=N, n_w=n_w, b_mn_major=True,
                     epi="store_bf16" if precision == 0 else "store_f32", precision=precision)
    torch.cuda.synchronize()
    ref = torch.stack([A[b].double() @ B[b % n_w].double() for b in range(nblk)])
    assert _rel(D, ref) < (2e-2 if precision == 0 else 1e-5)


@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("accumulate", [False, True])
def test_k_grouped_wgrad(precision, accumulate):
    ops = _ops()
    dt = torch.bfloat16 if precision == 0 else torch.float32
    nblk, rows, Mo, No, n_w = 6, 200, 192, 320, 3
    A = _rand(nblk, rows, Mo, dtype=dt)
    B = _rand(nblk, rows, No, dtype=dt)
    D0 = torch.randn(n_w, Mo, No, device="cuda")
    D = D0.clone()
    ops.grouped_gemm("k", A, B, D, nblk=nblk, rows=rows, Mo=Mo, No=No, n_w=n_w, epi="store_f32",
                     accumulate=accumulate, precision=precision)
    torch.cuda.synchronize()
    ref = torch.zeros(n_w, Mo, No, dtype=torch.float64, device="cuda")
    for b in range(nblk):
        ref[b % n_w] += A[b].double().T @ B[b].double()
    if accumulate:
        ref += D0.double()
    assert _rel(D, ref) < (5e-3 if precision == 0 else 1e-5)


def test_valid_rows_skip_and_kextent(gemm_ctas):
    ops = _ops()
    tile = 128 * int(gemm_ctas)
    nblk, rows, K, N = 4, 512, 128, 256
    valid = torch.tensor([0, 100, 512, 300], device="cuda", dtype=torch.int64)
    A = _rand(nblk, rows, K)
    for b in range(nblk):
        A[b, valid[b]:] = 0
    B = _rand(nblk, N, K, scale=K ** -0.5)
    D = torch.full((nblk, rows, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    ops.grouped_gemm("row", A, B, D, nblk=nblk, rows=rows, K=K, N=N, n_w=nblk, valid_rows=valid)
    torch.cuda.synchronize()
    for b in range(nblk):
        v = int(valid[b])
        vr = min((v + tile - 1) // tile * tile, rows)  # computed tiles cover whole row tiles
        ref = A[b, :vr].double() @ B[b].double().T
        if vr:
            assert _rel(D[b, :vr], ref) < 2e-2
        if vr < rows:
            assert torch.isnan(D[b, vr:].float()).all()  # skipped tiles untouched
    # wgrad over the same blocks: K extent = valid rows
    G = _rand(nblk, rows, N)
    W = torch.zeros(nblk, K, N, device="cuda")
    ops.grouped_gemm("k", A, G, W, nblk=nblk, rows=rows, Mo=K, No=N, n_w=nblk, epi="store_f32",
                     valid_rows=valid)
    torch.cuda.synchronize()
    for b in range(nblk):
        v = int(valid[b])
        ref = A[b, :v].double().T @ G[b, :v].double()
        if v == 0:
            assert W[b].abs().max().item() == 0
        else:
            assert _rel(W[b], ref) < 5e-3


def test_gelu_epilogues():
    ops = _ops()
    nblk, rows, K, H = 2, 256, 256, 512
    X = _rand(nblk, rows, K)
    W1 = _rand(nblk, H, K, scale=K ** -0.5)
    Z = torch.empty(nblk, rows, H, device="cuda", dtype=torch.bfloat16)
    Hh = torch.empty_like(Z)
    ops.grouped_gemm("row", X, W1, Z, nblk=nblk, rows=rows, K=K, N=H, n_w=nblk, epi="gelu_fwd",
                     D2=Hh, ldd2=H)
    torch.cuda.synchronize()
    zref = torch.stack([X[b].float() @ W1[b].float().T for b in range(nblk)])
    zb = zref.bfloat16().float().requires_grad_(True)
    href = F.gelu(zb)
    gref = torch.autograd.grad(href, zb, torch.ones_like(href))[0]
    # Z holds the saved derivative gelu'(Z), Hh = gelu(Z)
    assert _rel(Z, gref) < 1e-2
    assert _rel(Hh, href.detach()) < 1e-2
    # backward epilogue: dZ = (dO . W2^T) * gelu'(Z), W2 stored [w][M][H] (MN-major B)
    M = 256
    dO = _rand(nblk, rows, M)
    W2 = _rand(nblk, M, H, scale=M ** -0.5)
    dZ = torch.empty(nblk, rows, H, device="cuda", dtype=torch.bfloat16)
    ops.grouped_gemm("row", dO, W2, dZ, nblk=nblk, rows=rows, K=M, N=H, n_w=nblk, b_mn_major=True,
                     epi="gelu_bwd", Zin=Z, ldz=H)
    torch.cuda.synchronize()
    g = torch.stack([dO[b].float() @ W2[b].float() for b in range(nblk)]) * gref
    assert _rel(dZ, g) < 2e-2


def test_row_scatter_epilogue():
    """Row scatter (the N = 1 top-1 combine fused into GEMM2 / dgrad1): output
    row r lands in row map[r] of the target, bit-identical to the plain store;
    rows mapped to -1 and target rows nobody maps to stay untouched."""
    ops = _ops()
    torch.manual_seed(2)
    nblk, rows, K, N = 3, 300, 256, 320
    A = _rand(nblk, rows, K)
    B = _rand(nblk, N, K, scale=K ** -0.5)
    D = torch.empty(nblk, rows, N, device="cuda", dtype=torch.bfloat16)
    ops.grouped_gemm("row", A, B, D, nblk=nblk, rows=rows, K=K, N=N, n_w=nblk)
    T = nblk * rows + 50
    perm = torch.randperm(T, device="cuda")[: nblk * rows].to(torch.int32)
    perm[::7] = -1
    out = torch.full((T, N), 7.0, device="cuda", dtype=torch.bfloat16)
    ops.grouped_gemm("row", A, B, None, nblk=nblk, rows=rows, K=K, N=N, n_w=nblk, scatter_rows=perm,
                     scatter_out=out)
    torch.cuda.synchronize()
    flat = D.reshape(-1, N)
    keep = perm >= 0
    assert torch.equal(out[perm[keep].long()], flat[keep])
    untouched = torch.ones(T, dtype=torch.bool, device="cuda")
    untouched[perm[keep].long()] = False
    assert bool((out[untouched] == 7.0).all())


@pytest.mark.parametrize("inplace", [True, False])
def test_add_bf16_epilogue(inplace):
    """D = bf16(acc + Zin): exact on integer-valued operands (every product,
    sum and the final add are exact), in place (Zin = D, the gate backward's
    dx accumulation) and out of place, ragged rows."""
    ops = _ops()
    torch.manual_seed(1)
    nblk, rows, K, N = 2, 300, 64, 320
    A = torch.randint(-4, 5, (nblk, rows, K), device="cuda").to(torch.bfloat16)
    B = torch.randint(-4, 5, (nblk, N, K), device="cuda").to(torch.bfloat16)
    Z0 = torch.randint(-64, 65, (nblk, rows, N), device="cuda").to(torch.bfloat16)
    Z = Z0.clone()
    D = Z if inplace else torch.empty_like(Z)
    ops.grouped_gemm("row", A, B, D, nblk=nblk, rows=rows, K=K, N=N, n_w=nblk, epi="add_bf16",
                     Zin=Z, ldz=N)
    torch.cuda.synchronize()
    ref = (torch.stack([A[b].float() @ B[b].float().T for b in range(nblk)]) + Z0.float()).bfloat16()
    assert torch.equal(D, ref)
    if not inplace:
        assert torch.equal(Z, Z0)
    # random operands: within bf16 rounding of the fp32 result
    A = _rand(nblk, rows, K)
    B = _rand(nblk, N, K, scale=K ** -0.5)
    Z0 = _rand(nblk, rows, N)
    D = Z0.clone()
    ops.grouped_gemm("row", A, B, D, nblk=nblk, rows=rows, K=K, N=N, n_w=nblk, epi="add_bf16",
                     Zin=D, ldz=N)
    torch.cuda.synchronize()
    ref = torch.stack([A[b].float() @ B[b].float().T for b in range(nblk)]) + Z0.float()
    assert _rel(D, ref) < 1e-2


@pytest.mark.parametrize("H", [256, 640])
def test_swiglu_epilogues(H):
    ops = _ops()
    nblk, rows, K = 2, 256, 256
    X = _rand(nblk, rows, K)
    W1 = _rand(nblk, 2 * H, K, scale=K ** -0.5)  # interleaved [gate128 | up128] blocks
    Z = torch.empty(nblk, rows, 2 * H, device="cuda", dtype=torch.bfloat16)
    Hh = torch.empty(nblk, rows, H, device="cuda", dtype=torch.bfloat16)
    ops.grouped_gemm("row", X, W1, Z, nblk=nblk, rows=rows, K=K, N=2 * H, n_w=nblk,
                     epi="swiglu_fwd", D2=Hh, ldd2=H)
    torch.cuda.synchronize()
    zref = torch.stack([X[b].float() @ W1[b].float().T for b in range(nblk)])
    assert _rel(Z, zref) < 2e-2
    zb = Z.float().view(nblk, rows, H // 128, 2, 128)
    g, u = zb[:, :, :, 0, :].reshape(nblk, rows, H), zb[:, :, :, 1, :].reshape(nblk, rows, H)
    assert _rel(Hh, F.silu(g) * u) < 2e-2
    M = 256
    dO = _rand(nblk, rows, M)
    W2 = _rand(nblk, M, H, scale=M ** -0.5)
    dZ = torch.empty(nblk, rows, 2 * H, device="cuda", dtype=torch.bfloat16)
    ops.grouped_gemm("row", dO, W2, dZ, nblk=nblk, rows=rows, K=M, N=H, n_w=nblk, b_mn_major=True,
                     epi="swiglu_bwd", Zin=Z, ldz=2 * H, ldd=2 * H)
    torch.cuda.synchronize()
    gg, uu = g.clone().requires_grad_(True), u.clone().requires_grad_(True)
    dH = torch.stack([dO[b].float() @ W2[b].float() for b in range(nblk)])
    dg, du = torch.autograd.grad(F.silu(gg) * uu, (gg, uu), dH)
    dzb = dZ.float().view(nblk, rows, H // 128, 2, 128)
    assert _rel(dzb[:, :, :, 0, :].reshape(nblk, rows, H), dg) < 2e-2
    assert _rel(dzb[:, :, :, 1, :].reshape(nblk, rows, H), du) < 2e-2


def test_large_perf_smoke():
    """One C2-shaped forward GEMM; also reports achieved TFLOP/s."""
    ops = _ops()
    E, C, M, H = 16, 1024, 1024, 4096
    X = _rand(E, C, M)
    W1 = _rand(E, H, M, scale=M ** -0.5)
    Z = torch.empty(E, C, H, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=H, n_w=E)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    n = 10
    for _ in range(n):
        ops.grouped_gemm("row", X, W1, Z, nblk=E, rows=C, K=M, N=H, n_w=E)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    tflops = 2 * E * C * M * H / ms / 1e9
    print(f"\n[gemm] E{E} C{C} M{M} H{H}: {ms*1e3:.1f} us  {tflops:.0f} TFLOP/s")
    ref = X[3].float() @ W1[3].float().T
    assert _rel(Z[3], ref) < 2e-2


@pytest.mark.parametrize("kind", ["row", "k"])
def test_row_window_chunks(kind):
    """Pipeline chunks: rows [row0, row0+rows) of blocks holding rows_total rows."""
    ops = _ops()
    nblk, C, K, N = 4, 640, 256, 512
    A = _rand(nblk, C, K)
    if kind == "row":
        B = _rand(nblk, N, K, scale=K ** -0.5)
        D = torch.full((nblk, C, N), float("nan"), device="cuda", dtype=torch.bfloat16)
        for lo, hi in [(0, 256), (256, 512), (512, 640)]:
            ops.grouped_gemm("row", A, B, D, nblk=nblk, rows=hi - lo, rows_total=C, row0=lo, K=K,
                             N=N, n_w=nblk)
        torch.cuda.synchronize()
        ref = torch.stack([A[b].double() @ B[b].double().T for b in range(nblk)])
        assert _rel(D, ref) < 2e-2
    else:
        G = _rand(nblk, C, N)
        W = torch.zeros(2, K, N, device="cuda")
        for i, (lo, hi) in enumerate([(0, 256), (256, 512), (512, 640)]):
            ops.grouped_gemm("k", A, G, W, nblk=nblk, rows=hi - lo, rows_total=C, row0=lo, Mo=K,
                             No=N, n_w=2, epi="store_f32", accumulate=i > 0)
        torch.cuda.synchronize()
        ref = torch.zeros(2, K, N, dtype=torch.float64, device="cuda")
        for b in range(nblk):
            ref[b % 2] += A[b].double().T @ G[b].double()
        assert _rel(W, ref) < 5e-3


def test_two_devices_one_process(gemm_ctas):
    """Kernel attributes (dynamic shared memory) are per device: a process
    that drives two GPUs must get correct GEMMs and row moves on both."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    ops = _ops()
    E, C, K, N = 4, 256, 256, 512
    for dev in (0, 1):
        with torch.cuda.device(dev):
            X = (torch.randn(E, C, K, device="cuda")).to(torch.bfloat16)
            W = (torch.randn(E, N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
            Z = torch.empty(E, C, N, device="cuda", dtype=torch.bfloat16)
            ops.grouped_gemm("row", X, W, Z, nblk=E, rows=C, K=K, N=N, n_w=E)
            idx = torch.randperm(E * C, device="cuda").to(torch.int32)
            idx[::7] = -1
            src = X.view(E * C, K)
            out = ops.gather_rows(src, idx)
            torch.cuda.synchronize()
            ref = torch.stack([X[b].float() @ W[b].float().T for b in range(E)])
            assert _rel(Z, ref) < 2e-2
            keep = idx >= 0
            assert torch.equal(out[keep], src[idx[keep].long()])
            assert int(out[~keep].abs().sum()) == 0
