#!/usr/bin/env python
"""bench.py — FSMoE MoE-layer forward+backward throughput on B200.

Headline (BASELINE.json "metric"): MoE layer fwd+bwd tokens/sec at 1/2/4/8
B200 and the fraction of the GEMM / NVLink roofline.

Workload (default: BASELINE configs[2], the north-star Mixtral-8x7B shape):
per GPU 32768 tokens, d_model 4096, d_ffn 14336 SwiGLU (3 GEMMs), 8 experts
top-2 GShard routing (the reference's noisy_topk, k = 2), capacity factor 1.0
(C = 8192 per expert and rank), bf16 activations / expert weights with fp32
accumulation, fp64-exact gate. N GPUs = expert parallel over N ranks (8/N
experts each; N = 8 is one expert per GPU, N = 1 runs all 8 experts locally,
i.e. the same per-GPU expert work as the 8-GPU job), tokens per GPU fixed
(weak scaling). `--config gpt2m` runs configs[1] (GPT-2-medium shape, 16
experts top-1 Switch), `--config gpt2xl --gate G` SURVEY C5; the default run
also measures configs[1] at the same N as an extra key.

A step = gate -> order -> AlltoAll -> expert FFN -> AlltoAll -> I-order and
the full backward (expert dgrad + wgrad, combine/dispatch backward, gate
backward, gate-gradient allreduce), all inside libfsmoe.so / libfsmoe_cuda.so.

Usage:  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
        torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE layer fwd+bwd tokens/sec at 1/2/4/8 B200; % of GEMM/NVLink roofline"
WORKLOADS = {
    # configs[1] (the extra key; round 1's headline): EP over 2/4/8 with fixed tokens per GPU
    "gpt2m": dict(workload="gpt2-medium-shape MoE layer (BASELINE configs[1])", tokens_per_gpu=16384,
                  d_model=1024, d_ffn=4096, experts=16, top_k=1, gate="noisy_topk (Switch top-1)",
                  ffn="simple (GELU)", capacity_factor=1.0, dtype="bf16 / fp32 accumulate",
                  l2="inputs and activations larger than L2 (126 MB): no flush needed"),
    # configs[2], the headline: Mixtral-8x7B-shape layer, 32k tokens per GPU, 8 experts top-2
    # SwiGLU; on N GPUs each rank holds 8/N experts (N = 8: one expert per GPU;
    # N = 1 runs the same per-GPU expert GEMM work with all 8 experts local)
    "mixtral": dict(workload="Mixtral-8x7B-shape MoE layer (BASELINE configs[2])", tokens_per_gpu=32768,
                    d_model=4096, d_ffn=14336, experts=8, top_k=2, gate="noisy_topk (GShard top-2)",
                    ffn="gated3 (SwiGLU)", capacity_factor=1.0, dtype="bf16 / fp32 accumulate",
                    l2="inputs and activations larger than L2 (126 MB): no flush needed"),
    # GPT-2-XL-shape layer for the other gates (--gate), 4096
    # tokens per GPU (B 4 x L 1024), 8 experts top-2, C = 1024
    "gpt2xl": dict(workload="GPT-2-XL-shape MoE layer (SURVEY C5)", tokens_per_gpu=4096, d_model=1600,
                   d_ffn=6400, experts=8, top_k=2, gate="noisy_topk", ffn="simple (GELU)",
                   capacity_factor=1.0, dtype="bf16 / fp32 accumulate",
                   l2="weights + activations ~0.3 GB per step (> L2): no flush needed"),
}
WORKLOAD = WORKLOADS["mixtral"]
GATES = ("noisy_topk", "sigmoid_topk", "cosine_topk", "expert_choice")
NVLINK_GBS = 900.0  # nominal per direction per GPU (measured peer copy ~770)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ----------------------------------------------------------------- clocks --

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        """Start sampling and return once nvidia-smi is producing lines (its
        start-up takes a few hundred ms), so short timed regions get samples."""
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        self.n0 = 0
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20", "-i", str(self.gpu)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            t_end = time.time() + 5.0
            while time.time() < t_end and self._lines() < 1:
                time.sleep(0.02)
            self.n0 = self._lines()   # samples before the timed region are dropped
        except OSError:
            self.proc = None

    def _lines(self):
        with open(self.path) as f:
            return sum(1 for _ in f)

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if not self.proc:
            return out
        time.sleep(0.045)   # at least two more 20 ms samples cover the region's end
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            lines = f.readlines()
        for line in lines[self.n0:] if len(lines) > self.n0 else lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
            try:  # the full event-reason mask (nvml bit order) for the rest
                mask = int(parts[4], 16)
            except ValueError:
                mask = 0
            for bit, n in ((0x1, "gpu_idle"), (0x2, "applications_clocks_setting"), (0x10, "sync_boost"),
                           (0x80, "hw_power_brake_slowdown"), (0x100, "display_clock_setting")):
                if mask & bit:
                    reasons.add(n)
        os.unlink(self.path)
        if sm:
            out.update(sm_mhz=statistics.median(sm), sm_max_mhz=max(mx), reasons=sorted(reasons),
                       samples=len(sm))
        return out


# ------------------------------------------------------------ CPU baseline --

def cpu_threads_for(T, M, E, cap):
    """Threads that can each run one full routing instance at once: every
    reference call holds about x + 2 buffers + y in fp64 plus its copies
    (≈ 2.5·(E·C + T)·M·8 bytes); use at most 60 % of the available memory."""
    per = 2.5 * (E * cap + T) * M * 8
    avail = None
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    avail = int(line.split()[1]) * 1024
    except OSError:
        pass
    cores = os.cpu_count() or 1
    if not avail:
        return 1
    return int(max(1, min(cores, (0.6 * avail) // per)))


def cpu_layer_restatement(M, H, gated, top_k, threads, tokens=256):
    """The whole layer step on the host cores, for scale: a torch-CPU fp32
    restatement (NOT the reference, which has no FFN or backward) of the
    expert FFN forward + backward that every token runs top_k times (the
    dominant cost; gate and permutations are timed by cpu_baseline). A
    bounded sample: `tokens` tokens through top_k experts of the workload's
    shape, fwd + bwd with autograd, best of 2. Returns (tokens/s, seconds)."""
    import torch
    torch.set_num_threads(threads)
    g = torch.Generator().manual_seed(5)
    n1 = 2 * H if gated else H
    x = torch.rand(tokens, M, generator=g) * 2 - 1
    ws = [((torch.rand(n1, M, generator=g) * 2 - 1) / M ** 0.5).requires_grad_(True) for _ in range(top_k)]
    w2 = [((torch.rand(M, H, generator=g) * 2 - 1) / H ** 0.5).requires_grad_(True) for _ in range(top_k)]
    dy = torch.rand(tokens, M, generator=g) * 2 - 1
    best = None
    for _ in range(2):
        t0 = time.perf_counter()
        xi = x.clone().requires_grad_(True)
        y = 0
        for e in range(top_k):
            z = xi @ ws[e].T
            h = torch.nn.functional.silu(z[:, :H]) * z[:, H:] if gated else torch.nn.functional.gelu(z)
            y = y + h @ w2[e].T
        y.backward(dy)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return tokens / best, best


def cpu_reference_pass(threads, x, w_gate, w_noise, experts, top_k, capacity):
    """The reference's own implementation of the path (run_gate -> dispatch_tokens
    -> combine_tokens, fp64, identity experts; proj/src/workload.cpp:143-282)
    on host cores, over the SAME routing instance the GPU arm runs (all T
    tokens of one rank, capacity C): oracle/_ref (compiled from
    /root/reference) when present, else the C restatement. Every thread runs
    the whole instance once (the reference is serial per call; threads add
    throughput, not a split of the instance, which would change the capacity
    semantics). Returns (tokens/s, kind, threads, wall seconds)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    kind = "reference" if pyoracle.available("reference") else "port"
    orcs = [pyoracle.Oracle(kind) for _ in range(threads)]
    errs = []

    def work(i):
        try:
            o = orcs[i]
            g = o.run_gate("noisy_topk", top_k, 7, x, w_gate, w_noise)
            d = o.dispatch(x, experts, g.token, g.expert, capacity)
            o.combine(d.buffers, x.shape[0], experts, g.token, g.expert, g.weight, d.slot_of_pick,
                      x.shape[1])
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    wall = time.perf_counter() - t0
    if errs:
        raise errs[0]
    return threads * x.shape[0] / wall, kind, threads, wall


def cpu_inputs(tokens, M, E, seed=1):
    """The routing instance on the host: x (bf16 values, upcast to fp64, as the
    GPU arm's tokens), score and noise weights U(-1/sqrt(M), 1/sqrt(M))."""
    import numpy as np
    import torch
    rng = np.random.default_rng(seed)
    x = torch.from_numpy(rng.standard_normal((tokens, M), dtype=np.float32)).to(torch.bfloat16)
    x = x.double().numpy()
    wg = rng.uniform(-1, 1, (M, E)) / np.sqrt(M)
    wn = rng.uniform(-1, 1, (M, E)) / np.sqrt(M)
    return x, wg, wn


def instance_capacity():
    """capacity_tokens (workload.cpp:43-51) of the GPU arm's per-rank instance."""
    import math
    W = WORKLOAD
    return int(math.ceil(W["top_k"] * W["capacity_factor"] * W["tokens_per_gpu"] / W["experts"] - 1e-9))


def reference_arm(args):
    """--impl reference: the reference's CPU implementation of the path on the
    GPU arm's routing instance (T tokens, capacity C), all the threads the
    host's memory allows, each step = every thread routing the full instance."""
    M, E, T, k = WORKLOAD["d_model"], WORKLOAD["experts"], WORKLOAD["tokens_per_gpu"], WORKLOAD["top_k"]
    cap = instance_capacity()
    threads = cpu_threads_for(T, M, E, cap)
    x, wg, wn = cpu_inputs(T, M, E)
    # CPU warm-up: one pass (page-in, allocator); the GPU arm's W >= 3 rule is
    # about clocks and caches that a CPU pass does not have
    t_full = None
    for _ in range(max(min(args.warmup, 1), 1)):
        _, _, _, t_full = cpu_reference_pass(threads, x, wg, wn, E, k, cap)
    # bounded steps: the whole K-step run stays within ~4 minutes -- when K
    # full instances would not, every step routes a leading sub-instance of
    # T_s tokens (capacity recomputed for it at the same factor; the
    # reference's cost is linear in the tokens, so tokens/s is comparable)
    budget_s = 240.0
    T_s = T
    if t_full and args.steps * t_full > budget_s:
        T_s = max(1024, int(T * budget_s / (args.steps * t_full)) // 64 * 64)
    if T_s < T:
        import math
        cap = int(math.ceil(k * WORKLOAD["capacity_factor"] * T_s / E - 1e-9))
        x = x[:T_s]
    rates, walls, kind = [], [], "port"
    for _ in range(args.steps):
        r, kind, thr, wall = cpu_reference_pass(threads, x, wg, wn, E, k, cap)
        rates.append(r)
        walls.append(wall * 1e3)
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": min(args.warmup, 1),
        "ms_per_step": statistics.median(walls), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(WORKLOAD, capacity=cap,
                       reference_path="run_gate -> dispatch_tokens -> combine_tokens "
                       "(the reference has no expert FFN and no backward)"),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": kind,
                         "sample": (f"{threads} threads, each routing the GPU arm's full instance "
                                    f"(T {T}, d_model {M}, {E} experts, top-{k}, capacity {cap}) once per step"
                                    if T_s == T else
                                    f"{threads} threads, each routing the first {T_s} of the GPU arm's {T} "
                                    f"tokens (capacity {cap}) once per step, so {args.steps} steps fit "
                                    f"~{budget_s:.0f} s (a full instance takes {t_full:.1f} s)")},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------- GPU arm --

def gemm_roofline(layer, peaks, reps=5):
    """Time the step's six expert GEMM launches standalone (same shapes and
    buffers, full capacity rows) with CUDA events on the launching stream."""
    import torch
    from paper_2501_10714_b200 import ops
    cfg = layer.cfg
    M, H, N1 = cfg.model_dim, cfg.ffn_dim, layer.n1
    nblk, C, El = layer.world * layer.el, layer.capacity, layer.el
    bf = torch.bfloat16
    rows = nblk * C
    X = layer.buffer("X_recv", bf, (nblk, C, M))
    Z = layer.buffer("Z", bf, (nblk, C, N1))
    Hh = layer.buffer("H", bf, (nblk, C, H))
    O = torch.empty(nblk, C, M, device=layer.device, dtype=bf)
    dO = torch.randn(nblk, C, M, device=layer.device).to(bf)
    dX = torch.empty_like(O)
    gw1 = torch.empty(El, N1, M, device=layer.device)
    gw2 = torch.empty(El, M, H, device=layer.device)
    Zc = Z.clone()
    calls = [
        ("fwd1", 2 * rows * M * N1, lambda: ops.grouped_gemm(
            "row", X, layer.w1, Z, nblk=nblk, rows=C, K=M, N=N1, n_w=El,
            epi="gelu_fwd" if cfg.ffn == "simple" else "swiglu_fwd", D2=Hh, ldd2=H)),
        ("fwd2", 2 * rows * H * M, lambda: ops.grouped_gemm(
            "row", Hh, layer.w2, O, nblk=nblk, rows=C, K=H, N=M, n_w=El)),
        ("wgrad2", 2 * rows * M * H, lambda: ops.grouped_gemm(
            "k", dO, Hh, gw2, nblk=nblk, rows=C, Mo=M, No=H, n_w=El, epi="store_f32")),
        ("dgrad2", 2 * rows * M * H, lambda: ops.grouped_gemm(
            "row", dO, layer.w2, Zc, nblk=nblk, rows=C, K=M, N=H, n_w=El, b_mn_major=True,
            epi="gelu_bwd" if cfg.ffn == "simple" else "swiglu_bwd", Zin=Z, ldz=N1, ldd=N1)),
        ("wgrad1", 2 * rows * N1 * M, lambda: ops.grouped_gemm(
            "k", Zc, X, gw1, nblk=nblk, rows=C, Mo=N1, No=M, n_w=El, epi="store_f32")),
        ("dgrad1", 2 * rows * N1 * M, lambda: ops.grouped_gemm(
            "row", Zc, layer.w1, dX, nblk=nblk, rows=C, K=N1, N=M, n_w=El, b_mn_major=True)),
    ]
    # The six launches cycled in step order for >= 1.5 s (after 0.5 s of
    # warm-up), so the figure is the power-capped steady state the step runs
    # in (a few hundred ms of back-to-back GEMMs read ~5 % fast: the clocks
    # had not settled); per-launch split from events around each launch of
    # the last 10 sets.
    E_ = torch.cuda.Event
    s, e = E_(enable_timing=True), E_(enable_timing=True)
    for _, _, fn in calls:
        fn()
    torch.cuda.synchronize()
    s.record()
    for _, _, fn in calls:
        fn()
    e.record()
    torch.cuda.synchronize()
    set_ms = max(s.elapsed_time(e), 1e-3)
    for _ in range(int(500.0 / set_ms) + 1):
        for _, _, fn in calls:
            fn()
    nsets = max(reps, int(1500.0 / set_ms) + 1)
    s.record()
    for _ in range(nsets):
        for _, _, fn in calls:
            fn()
    e.record()
    tail = [[E_(enable_timing=True) for _ in range(len(calls) + 1)] for _ in range(10)]
    for evs in tail:
        evs[0].record()
        for i, (_, _, fn) in enumerate(calls):
            fn()
            evs[i + 1].record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / nsets
    per = {name: (flops, sum(evs[i].elapsed_time(evs[i + 1]) for evs in tail) / len(tail))
           for i, (name, flops, _) in enumerate(calls)}
    flops = sum(v[0] for v in per.values())
    achieved = flops / (ms * 1e-3) / 1e12
    # MEASURED_PEAKS.json: the burst cuBLAS figure for a kernel timed alone
    # (short), the sustained (4 s back-to-back) one for this power-capped run
    sustained = ms * nsets >= 50.0
    peak = peaks.get("bf16_tflops_sustained" if sustained else "bf16_tflops", 1590.0)
    epi = "SwiGLU" if cfg.ffn == "gated3" else "GELU"
    return {
        "bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
        "frac": round(achieved / peak, 4), "traffic": None,
        "frac_vs_burst": round(achieved / peaks.get("bf16_tflops", 1590.0), 4),
        "kernel": f"grouped_gemm_kernel (tcgen05 cta_group::2; 6 launches/step: fwd1 ({epi} epilogue), "
                  f"fwd2, wgrad2, dgrad2 ({epi} backward epilogue), wgrad1, dgrad1)",
        "flops_per_step": flops, "gemm_ms_per_step": round(ms, 4),
        "per_launch_ms": {k: round(v[1], 4) for k, v in per.items()},
        "peak_kind": ("bf16_tflops_sustained" if sustained else "bf16_tflops (burst)")
                     + f" of MEASURED_PEAKS.json (the six launches cycled {nsets} times = "
                       f"{ms * nsets:.0f} ms of GEMMs after 0.5 s warm-up)",
    }, flops, ms


def timeline_summary(trace: str, steps: int):
    """Per-phase device time (ms/step) from the layer's Chrome trace, plus how
    much of the comm stream's time is NOT hidden under compute (exposed)."""
    ev = json.loads(trace)["traceEvents"]
    per = {}
    comp, comm = [], []
    for x in ev:
        name = x["name"].split("[")[0]
        per[name] = per.get(name, 0.0) + x["dur"] / 1e3
        (comm if x["tid"] == 0 else comp).append((x["ts"], x["ts"] + x["dur"]))
    comp.sort()
    exposed = 0.0
    for a, b in comm:
        covered = 0.0
        for c, d in comp:
            lo, hi = max(a, c), min(b, d)
            if hi > lo:
                covered += hi - lo
        exposed += (b - a) - covered
    span = (max(b for _, b in comp + comm) - min(a for a, _ in comp + comm)) / 1e3
    return {"phase_ms_per_step": {k: round(v / steps, 4) for k, v in sorted(per.items())},
            "comm_ms_per_step": round(sum(b - a for a, b in comm) / 1e3 / steps, 4),
            "comm_exposed_ms_per_step": round(exposed / 1e3 / steps, 4),
            "traced_ms_per_step": round(span / steps, 4),
            "note": "traced run synchronises per phase call; shares, not absolute step time"}


def layer_config(W, gate=None, r_fwd=1, r_bwd=1, transport=""):
    from paper_2501_10714_b200.layer import MoEConfig
    gate = gate or W["gate"].split()[0]
    # expert choice: every expert takes C = k f T / E tokens (workload.cpp:156-171,
    # the layer derives C from k); cosine: a 64-row projection (the reference
    # leaves the dimension open)
    return MoEConfig(tokens=W["tokens_per_gpu"], model_dim=W["d_model"], ffn_dim=W["d_ffn"],
                     experts=W["experts"], top_k=W["top_k"], gate=gate, ffn=W["ffn"].split()[0],
                     capacity_factor=W["capacity_factor"], proj_dim=64 if gate == "cosine_topk" else 0,
                     precision="bf16", seed=7, r_fwd=r_fwd, r_bwd=r_bwd, transport=transport)


def make_layer(W, args, world, rank, ep, gate=None, pipe=None):
    from paper_2501_10714_b200.layer import MoELayer
    rf, rb, tr = pipe or (max(args.r_fwd, 1), max(args.r_bwd, 1), args.transport)
    return MoELayer(layer_config(W, gate, rf, rb, tr), ep, init_seed=1)


def choose_pipeline(W, args, world, rank, ep, gate, x, dy):
    """FSMoE's online profiling on this box (paper_2501_10714_b200.autotune):
    collectives + GEMM chunks -> bench CSV -> fit_profile -> plan_layer (the
    reference's planner), then the plan and its neighbours measured on the
    real layer for each EP transport; the fastest is used. Explicit
    --r-fwd / --r-bwd / --transport skip it. Returns ((r_fwd, r_bwd,
    transport), report)."""
    if world == 1:
        return (max(args.r_fwd, 1), max(args.r_bwd, 1), args.transport), {"how": "N = 1: no exchange, r = 1"}
    if args.r_fwd > 0 and args.r_bwd > 0:
        return (args.r_fwd, args.r_bwd, args.transport), {"how": "given on the command line"}
    from paper_2501_10714_b200 import autotune
    cfg = layer_config(W, gate)
    samples, _ = autotune.collect(cfg, world, r_max=4)
    p = autotune.plan(cfg, samples, world, r_max=4)
    trs = (args.transport,) if args.transport else ("peer", "ce")
    rf, rb, meas = autotune.refine(cfg, ep, (p["r_fwd"], p["r_bwd"]), x, dy, r_max=4, steps=5, transports=trs)
    rep = {"how": "on-box profile -> fit_profile -> plan_layer -> refined on the layer (autotune.refine)",
           "planned": [p["r_fwd"], p["r_bwd"]], "chosen": [rf, rb, cfg.transport],
           "refine_ms": {f"{k[0]}:r{k[1]}": round(v, 4) for k, v in meas.items()}}
    return (rf, rb, cfg.transport), rep


def timed_steps(layer, x, y, dy, dx, args, world, warm_seconds):
    """W warm-up steps, then more until `warm_seconds` of steady stepping have
    passed (clocks settle under the power cap), then EXACTLY args.steps timed
    steps between barriers + synchronize, CUDA events on the launching stream,
    max over ranks. Returns (ms/step, extra warm-up steps, clocks, launches,
    exposed-wait ms/step of this rank)."""
    import ctypes
    import torch
    import torch.distributed as dist
    from paper_2501_10714_b200 import _native
    for _ in range(args.warmup):
        layer.forward(x, y)
        layer.backward(dy, dx)
    torch.cuda.synchronize()
    extra = 0
    t_end = time.perf_counter() + warm_seconds
    while time.perf_counter() < t_end:
        layer.forward(x, y)
        layer.backward(dy, dx)
        torch.cuda.synchronize()
        extra += 1
    if world > 1:
        dist.barrier()
    lib = _native.cuda_lib()
    lib.fsmoe_launch_count.restype = ctypes.c_longlong
    wait_buf = layer.buffer("wait_ns", torch.int64) if world > 1 else None
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clocks.start()
    w0 = int(layer.buffer("wait_ns", torch.int64).item()) if world > 1 else 0
    n0 = lib.fsmoe_launch_count()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s.record()
    for _ in range(args.steps):
        layer.forward(x, y)
        layer.backward(dy, dx)
    e.record()
    torch.cuda.synchronize()
    launches = lib.fsmoe_launch_count() - n0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = s.elapsed_time(e) / args.steps
    wait_ms = 0.0
    if wait_buf is not None:
        wait_ms = (int(layer.buffer("wait_ns", torch.int64).item()) - w0) / 1e6 / args.steps
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), extra, clk, launches, wait_ms


def gpu_arm(args):
    import torch
    import torch.distributed as dist
    from paper_2501_10714_b200.layer import EpGroup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks, peak_kind = load_peaks()
    T, M, H, E = (WORKLOAD["tokens_per_gpu"], WORKLOAD["d_model"], WORKLOAD["d_ffn"],
                  WORKLOAD["experts"])
    gate = args.gate or WORKLOAD["gate"].split()[0]
    ep = EpGroup(world, rank, local, max_ctas=args.nccl_ctas) if world > 1 else None
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    x = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    dx = torch.empty_like(x)
    y = torch.empty_like(x)
    try:
        pipe, pipe_rep = choose_pipeline(WORKLOAD, args, world, rank, ep, gate, x, dy)
    except Exception as exc:  # the planning step only picks r / transport: fall back to r = 1
        pipe, pipe_rep = (1, 1, args.transport), {"how": f"planning failed ({exc!r}); r = 1"}
        torch.cuda.synchronize()
    layer = make_layer(WORKLOAD, args, world, rank, ep, gate, pipe=pipe)
    ms, extra_warm, clk, launches, wait_ms = timed_steps(layer, x, y, dy, dx, args, world,
                                                         args.warm_seconds)
    value = world * T / (ms * 1e-3)
    # exposed AlltoAll (untraced): the time each rank's compute stream spent
    # spinning on peer arrival flags inside the timed steps (globaltimer in
    # peer_wait_kernel), max over ranks
    exposed = None
    if world > 1:
        per = [None] * world
        dist.all_gather_object(per, wait_ms)
        exposed = {"ms_per_step": max(per), "frac_of_step": max(per) / ms,
                   "by_rank_ms_per_step": per,
                   "how": "per-rank peer-flag wait time (globaltimer in peer_wait_kernel) over the "
                          "timed steps, untraced; max over ranks"}

    # e2e: host (pinned) inputs in, the step's results out, through the public
    # layer API. Every step copies its x and dy host->device and reads y and
    # dx back device->host inside the timed region; the copies run on their
    # own streams (copy engines), triple-buffered against the previous / next
    # step's compute, the way a training loop feeds a layer.
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        dyh = dy.cpu().pin_memory()
        NB = 3  # triple-buffered: step i+1's H2D never waits on step i-1's D2H
        yh = [torch.empty_like(xh).pin_memory() for _ in range(NB)]
        dxh = [torch.empty_like(xh).pin_memory() for _ in range(NB)]
        xd = [torch.empty_like(x) for _ in range(NB)]
        dyd = [torch.empty_like(dy) for _ in range(NB)]
        yd = [torch.empty_like(x) for _ in range(NB)]
        dxd = [torch.empty_like(dx) for _ in range(NB)]
        comp = torch.cuda.current_stream()
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ev_x = [torch.cuda.Event() for _ in range(NB)]
        ev_dy = [torch.cuda.Event() for _ in range(NB)]
        ev_y = [torch.cuda.Event() for _ in range(NB)]
        ev_done = [torch.cuda.Event() for _ in range(NB)]
        ev_free = [torch.cuda.Event() for _ in range(NB)]
        for i in range(NB):
            ev_free[i].record(comp)

        def e2e_steps(n):
            for i in range(n):
                b = i % NB
                with torch.cuda.stream(s_in):
                    s_in.wait_event(ev_free[b])       # step i-NB no longer uses set b
                    xd[b].copy_(xh, non_blocking=True)
                    ev_x[b].record(s_in)
                    dyd[b].copy_(dyh, non_blocking=True)
                    ev_dy[b].record(s_in)
                comp.wait_event(ev_x[b])              # forward needs x only
                layer.forward(xd[b], yd[b])
                ev_y[b].record(comp)
                comp.wait_event(ev_dy[b])
                layer.backward(dyd[b], dxd[b])
                ev_done[b].record(comp)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev_y[b])         # y leaves while the backward runs
                    yh[b].copy_(yd[b], non_blocking=True)
                    s_out.wait_event(ev_done[b])
                    dxh[b].copy_(dxd[b], non_blocking=True)
                    ev_free[b].record(s_out)        # results read out, inputs consumed
            comp.wait_stream(s_out)

        # >= 50 steps: the copy pipeline's fill (first step's inputs) and drain (last
        # step's outputs) are inside the timed region and amortise over the run
        ke = max(args.steps, 50)
        e2e_steps(NB)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        e2e_steps(ke)
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / ke], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
        e2e = {"value": world * T / (ems * 1e-3), "unit": "tokens/s",
               "h2d_bytes_per_step": 2 * x.numel() * x.element_size(),
               "d2h_bytes_per_step": 2 * x.numel() * x.element_size(), "ms_per_step": ems,
               "steps": ke,
               "api": "paper_2501_10714_b200.layer.MoELayer forward+backward (libfsmoe.so C ABI)",
               "copies": "pinned host x and dy in, the whole y and dx out, every step, on copy "
                         "streams triple-buffered against compute, all inside the timed region"}

    timeline = None
    if args.trace or (world > 1 and not args.no_timeline):
        # measured per-phase timeline (3 extra steps, outside the timed
        # region; tracing synchronises per phase): shares, not step time
        nt = 3
        layer.set_trace(True)
        for _ in range(nt):
            layer.forward(x, y)
            layer.backward(dy, dx)
        torch.cuda.synchronize()
        tj = layer.trace_json()
        layer.set_trace(False)
        if args.trace:
            os.makedirs(os.path.dirname(os.path.abspath(args.trace)) or ".", exist_ok=True)
            with open(f"{args.trace}.rank{rank}.json", "w") as f:
                f.write(tj)
        timeline = timeline_summary(tj, nt)

    roof, gflops, gms = gemm_roofline(layer, peaks)
    roof["peak_source"] = peak_kind
    traffic_file = os.path.join(ROOT, "profiles", f"gemm_traffic_{args.config}.json")
    if os.path.exists(traffic_file):
        with open(traffic_file) as f:
            roof["traffic"] = json.load(f).get("bytes_per_step")
            roof["traffic_source"] = os.path.relpath(traffic_file, ROOT)
    # step roofline (north star): max(GEMM flops at peak, AlltoAll bytes at NVLink)
    C = layer.capacity
    a2a_bytes = 4 * E * C * M * 2 * (world - 1) / world
    pk = peaks.get("bf16_tflops_sustained" if ms >= 10.0 else "bf16_tflops", 1590.0)
    t_gemm = gflops / (pk * 1e12) * 1e3
    t_a2a = a2a_bytes / (NVLINK_GBS * 1e9) * 1e3
    a2a_meas = None
    if world > 1:
        # what NCCL's AlltoAll moves on this box for the step's volume (one
        # exchange = a quarter of the step's a2a bytes), beside the 900 GB/s
        # nominal the roofline uses
        n = E * C * M // world * world
        sb = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        rb = torch.empty_like(sb)
        for _ in range(3):
            dist.all_to_all_single(rb, sb)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            dist.all_to_all_single(rb, sb)
        e.record()
        torch.cuda.synchronize()
        ams = s.elapsed_time(e) / 10
        tt = torch.tensor([ams], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ams = float(tt.item())
        moved = n * 2 * (world - 1) / world
        a2a_meas = {"nccl_alltoall_ms": ams, "bytes_out_per_gpu": moved,
                    "busbw_gbs": moved / (ams * 1e-3) / 1e9,
                    "note": "torch.distributed all_to_all_single (NCCL) of one dispatch's volume"}
        del sb, rb
    step_roof = {"gemm_flops": gflops, "a2a_bytes_out_per_gpu": a2a_bytes,
                 "a2a_measured": a2a_meas, "peak_tflops": pk,
                 "peak_kind": "bf16_tflops_sustained" if ms >= 10.0 else "bf16_tflops (burst)",
                 "roofline_ms": max(t_gemm, t_a2a), "measured_ms": ms,
                 "frac": max(t_gemm, t_a2a) / ms, "gemm_share_of_step": gms / ms,
                 "frac_vs_burst": max(gflops / (peaks.get("bf16_tflops", 1590.0) * 1e12) * 1e3,
                                      t_a2a) / ms,
                 "frac_vs_spec": max(gflops / 2.25e15 * 1e3, t_a2a) / ms,
                 "roofline_tokens_per_s": world * T / (max(t_gemm, t_a2a) * 1e-3)}
    # kept-row GEMM work of the last step (capacity drops and padding rows
    # excluded): rows every rank dispatched, averaged per GPU
    k_ = WORKLOAD["top_k"]
    kept = torch.tensor([float(T * k_ - int(layer.buffer("dropped", torch.int64).item()))],
                        device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(kept)
    kept_rows = float(kept.item()) / world
    g_ = 3 if "gated3" in WORKLOAD["ffn"] else 2
    kept_flops = 3 * g_ * 2 * kept_rows * M * WORKLOAD["d_ffn"]
    step_roof["kept_rows_per_gpu"] = kept_rows
    step_roof["capacity_rows_per_gpu"] = E * C
    step_roof["kept_row_gemm_flops"] = kept_flops
    step_roof["kept_row_frac"] = max(kept_flops / (pk * 1e12) * 1e3, t_a2a) / ms
    layer.close()
    del layer
    torch.cuda.empty_cache()

    # configs[1] at the same N (extra key; the headline line is configs[2])
    extra = None
    if args.config == "mixtral" and not args.no_extra:
        W1 = WORKLOADS["gpt2m"]
        T1, M1 = W1["tokens_per_gpu"], W1["d_model"]
        x1 = torch.randn(T1, M1, device="cuda", generator=g).to(torch.bfloat16)
        dy1 = torch.randn(T1, M1, device="cuda", generator=g).to(torch.bfloat16)
        try:
            pipe1, pipe1_rep = choose_pipeline(W1, args, world, rank, ep, None, x1, dy1)
        except Exception as exc:
            pipe1, pipe1_rep = (1, 1, args.transport), {"how": f"planning failed ({exc!r}); r = 1"}
        l1 = make_layer(W1, args, world, rank, ep, pipe=pipe1)
        # a ~1 ms step: time >= 1000 steps (about a second) after the same 3 s
        # warm-up as the headline, so the clocks are the power-capped steady
        # state, not a 20-step burst
        args1 = argparse.Namespace(**vars(args))
        args1.steps = max(args.steps, 1000)
        ms1, ex1, clk1, _, wait1 = timed_steps(l1, x1, torch.empty_like(x1), dy1, torch.empty_like(x1),
                                               args1, world, args.warm_seconds)
        extra = {"workload": W1["workload"], "value": world * T1 / (ms1 * 1e-3), "unit": "tokens/s",
                 "ms_per_step": ms1, "steps": args1.steps, "capacity": l1.capacity, "clocks": clk1,
                 "r_fwd": pipe1[0], "r_bwd": pipe1[1], "pipeline": pipe1_rep}
        try:  # its six expert GEMMs, timed the same way as the headline's
            roof1, _, _ = gemm_roofline(l1, peaks)
            extra["roofline"] = {k: roof1[k] for k in ("bound", "achieved", "peak", "unit", "frac",
                                                       "frac_vs_burst", "gemm_ms_per_step",
                                                       "per_launch_ms", "peak_kind")}
        except Exception as exc:  # noqa: BLE001 (a report beside the measurement)
            extra["roofline"] = {"unavailable": repr(exc)[:200]}
        if world > 1:
            per1 = [None] * world
            dist.all_gather_object(per1, wait1)
            extra["exposed_alltoall_ms_per_step"] = max(per1)
        l1.close()
        del l1

    cpu = None
    cpu_restatement = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cap = instance_capacity()
        thr = cpu_threads_for(T, M, E, cap)
        xs, wg, wn = cpu_inputs(T, M, E)
        rate, kind, thr, wall = cpu_reference_pass(thr, xs, wg, wn, E, WORKLOAD["top_k"], cap)
        cpu = {"value": rate, "unit": "tokens/s", "cores": thr, "kind": kind,
               "sample": f"{thr} threads, each routing this workload's full per-GPU instance (T {T}, "
                         f"d_model {M}, {E} experts, top-{WORKLOAD['top_k']}, capacity {cap}) once: "
                         f"run_gate->dispatch_tokens->combine_tokens in {wall:.1f} s; the reference "
                         "has no FFN/backward"}
        try:
            rr, rs = cpu_layer_restatement(M, WORKLOAD["d_ffn"], "gated3" in WORKLOAD["ffn"], WORKLOAD["top_k"], thr)
            cpu_restatement = {"value": rr, "unit": "tokens/s", "cores": thr,
                               "what": "torch-CPU fp32 restatement of the expert FFN forward + backward each "
                                       "token runs (top-k experts) -- a restatement, not the reference",
                               "sample": f"256 tokens x {WORKLOAD['top_k']} experts of the workload's shape, "
                                         f"best of 2: {rs:.2f} s"}
        except Exception as e:  # noqa: BLE001 (a report, not the measurement)
            cpu_restatement = {"unavailable": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random tokens, random-init experts)",
            "config": dict(WORKLOAD, parallelism=f"ep{world}", r_fwd=pipe[0], r_bwd=pipe[1],
                           transport=(pipe[2] or "peer") if world > 1 else None, pipeline=pipe_rep,
                           capacity=C, warmup_extra_steps=extra_warm,
                           warmup_note=f"W warm-up steps, then more until {args.warm_seconds:.0f} s "
                                       "of stepping (steady clocks)",
                           **({"gate": gate} if args.gate else {})),
            "clocks": clk, "e2e": e2e, "gpu_launches": launches,
            "roofline": roof, "step_roofline": step_roof, "cpu_baseline": cpu,
            "exposed_alltoall": exposed,
        }
        if cpu_restatement:
            line["cpu_restatement"] = cpu_restatement
        if extra:
            line["configs[1]"] = extra
        if timeline:
            line["timeline"] = timeline
        print(json.dumps(line), flush=True)
    if ep:
        ep.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--r-fwd", type=int, default=0, help="pipeline degree (0: FSMoE's online plan at N > 1)")
    ap.add_argument("--r-bwd", type=int, default=0)
    ap.add_argument("--transport", default="", choices=["", "peer", "ce", "nccl"],
                    help="EP exchange ('' = chosen with the pipeline degree, or FSMOE_EP_TRANSPORT)")
    ap.add_argument("--nccl-ctas", type=int, default=16)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the configs[1] extra measurement")
    ap.add_argument("--no-timeline", action="store_true", help="skip the traced per-phase timeline")
    ap.add_argument("--warm-seconds", type=float, default=3.0,
                    help="keep warming up (after W steps) until this much stepping has passed")
    ap.add_argument("--trace", default="", help="write per-rank measured timelines to PATH.rankN.json")
    ap.add_argument("--config", default="mixtral", choices=sorted(WORKLOADS),
                    help="mixtral = BASELINE configs[2] (the north-star headline); gpt2m = configs[1]; "
                         "gpt2xl = SURVEY C5 (use with --gate)")
    ap.add_argument("--gate", default=None, choices=GATES,
                    help="gate kind (default: the workload's, noisy_topk)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    global WORKLOAD
    WORKLOAD = WORKLOADS[args.config]
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        reference_arm(args)
        return
    gpu_arm(args)


if __name__ == "__main__":
    main()
