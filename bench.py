#!/usr/bin/env python
"""bench.py — FSMoE MoE-layer forward+backward throughput on B200.

Headline (BASELINE.json "metric"): MoE layer fwd+bwd tokens/sec at 1/2/4/8
B200 and the fraction of the GEMM / NVLink roofline.

Workload (BASELINE configs[1], the GPT-2-medium shape): per GPU 16384 tokens,
d_model 1024, d_ffn 4096 (simple FFN, GELU), 16 experts top-1 Switch routing
(the reference's noisy_topk with k=1: combine weight exactly 1.0), capacity
factor 1.0 (C = 1024 per expert and rank), bf16 activations / expert weights
with fp32 accumulation, fp64-exact gate. N GPUs = expert parallel over N ranks
(16/N experts each), tokens per GPU fixed (weak scaling).

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
    # the headline (configs[1]): fits one GPU, EP over 2/4/8 with fixed tokens per GPU
    "gpt2m": dict(workload="gpt2-medium-shape MoE layer (BASELINE configs[1])", tokens_per_gpu=16384,
                  d_model=1024, d_ffn=4096, experts=16, top_k=1, gate="noisy_topk (Switch top-1)",
                  ffn="simple (GELU)", capacity_factor=1.0, dtype="bf16 / fp32 accumulate",
                  l2="inputs and activations larger than L2 (126 MB): no flush needed"),
    # configs[2]: Mixtral-8x7B-shape layer, 32k tokens per GPU, 8 experts top-2
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
WORKLOAD = WORKLOADS["gpt2m"]
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

def cpu_reference_rate(seconds: float, threads: int, tokens_per_call: int, x, w_gate, w_noise,
                       experts: int, capacity_per_call: int):
    """The reference's own implementation of the path (run_gate -> dispatch_tokens
    -> combine_tokens, fp64, identity experts; proj/src/workload.cpp:143-282) on
    host cores: oracle/_ref (compiled from /root/reference) when present, else
    the C restatement. One call per thread on its own token shard, repeated
    until `seconds` elapse. Returns (tokens/s, kind, threads, calls)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    kind = "reference" if pyoracle.available("reference") else "port"
    orcs = [pyoracle.Oracle(kind) for _ in range(threads)]
    done = [0] * threads
    stop = [False]

    def work(i):
        o = orcs[i]
        while not stop[0]:
            xs = x[(i * tokens_per_call) % x.shape[0]:][:tokens_per_call]
            g = o.run_gate("noisy_topk", WORKLOAD["top_k"], 7, xs, w_gate, w_noise)
            d = o.dispatch(xs, experts, g.token, g.expert, capacity_per_call)
            o.combine(d.buffers, xs.shape[0], experts, g.token, g.expert, g.weight, d.slot_of_pick,
                      xs.shape[1])
            done[i] += 1

    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    time.sleep(seconds)
    stop[0] = True
    for t in ts:
        t.join()
    wall = time.perf_counter() - t0
    calls = sum(done)
    return calls * tokens_per_call / wall, kind, threads, calls, wall


def cpu_inputs(tokens, M, E, seed=1):
    import numpy as np
    rng = np.random.default_rng(seed)
    import torch
    x = torch.from_numpy(rng.uniform(-1, 1, (tokens, M))).to(torch.bfloat16).double().numpy()
    wg = rng.uniform(-1, 1, (M, E)) / np.sqrt(M)
    wn = rng.uniform(-1, 1, (M, E)) / np.sqrt(M)
    return x, wg, wn


def reference_arm(args):
    """--impl reference: the reference's CPU implementation of the path, timed
    with all host threads on this workload's shape, one bounded sample/step."""
    M, E, T = WORKLOAD["d_model"], WORKLOAD["experts"], 1024
    threads = os.cpu_count() or 1
    x, wg, wn = cpu_inputs(T * threads, M, E)
    cap = -(-T * WORKLOAD["top_k"] // E)  # capacity_tokens(k, f=1.0) for the sample's B*L
    for _ in range(args.warmup):
        cpu_reference_rate(0.2, threads, T, x, wg, wn, E, cap)
    rates, walls, kind = [], [], "port"
    for _ in range(args.steps):
        r, kind, thr, calls, wall = cpu_reference_rate(1.0, threads, T, x, wg, wn, E, cap)
        rates.append(r)
        walls.append(wall * 1e3 / max(calls / threads, 1))
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(walls), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(WORKLOAD, reference_path="run_gate -> dispatch_tokens -> combine_tokens "
                       "(the reference has no expert FFN and no backward)"),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": kind,
                         "sample": f"{threads} threads x {T} tokens per call, d_model {M}, "
                                   f"{E} experts, top-{WORKLOAD['top_k']}, ~1 s per step"},
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
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per = {}
    for name, flops, fn in calls:
        fn()
        torch.cuda.synchronize()
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        per[name] = (flops, s.elapsed_time(e) / reps)
    flops = sum(v[0] for v in per.values())
    ms = sum(v[1] for v in per.values())
    achieved = flops / (ms * 1e-3) / 1e12
    peak = peaks.get("bf16_tflops", 1590.0)
    return {
        "bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
        "frac": round(achieved / peak, 4), "traffic": None,
        "kernel": "grouped_gemm_kernel (tcgen05 cta_group::2; 6 launches/step: fwd1 (256x256 tiles, GELU) fwd2 wgrad2 (256x512) dgrad2 (256x256, GELU bwd) wgrad1 dgrad1 (256x512))",
        "flops_per_step": flops, "gemm_ms_per_step": round(ms, 4),
        "per_launch_ms": {k: round(v[1], 4) for k, v in per.items()},
        "peak_kind": "bf16_tflops (burst) of MEASURED_PEAKS.json",
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


def gpu_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2501_10714_b200 import _native
    from paper_2501_10714_b200.layer import EpGroup, MoEConfig, MoELayer

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
    # expert choice: every expert takes C = k f T / E tokens (workload.cpp:156-171,
    # the layer derives C from k); cosine: a 64-row projection (the reference
    # leaves the dimension open)
    cfg = MoEConfig(tokens=T, model_dim=M, ffn_dim=H, experts=E, top_k=WORKLOAD["top_k"], gate=gate, ffn=WORKLOAD["ffn"].split()[0], capacity_factor=1.0,
                    proj_dim=64 if gate == "cosine_topk" else 0,
                    precision="bf16", seed=7, r_fwd=args.r_fwd, r_bwd=args.r_bwd)
    ep = EpGroup(world, rank, local, max_ctas=args.nccl_ctas) if world > 1 else None
    layer = MoELayer(cfg, ep, init_seed=1)
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    x = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
    dx = torch.empty_like(x)
    y = torch.empty_like(x)
    for _ in range(args.warmup):
        layer.forward(x, y)
        layer.backward(dy, dx)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    lib = _native.cuda_lib()
    lib.fsmoe_launch_count.restype = __import__("ctypes").c_longlong
    clocks = ClockSampler(local)
    clocks.start()
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
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * T / (ms * 1e-3)

    # e2e: host (pinned) inputs in, the step's result out, through the public
    # layer API. Every step copies its x and dy host->device inside the timed
    # region and reads a metric of the step's result back (a checksum of dx,
    # 4 bytes — the contract's "loss or metric"); the copies run on their own
    # streams (copy engines), triple-buffered against the previous / next
    # step's compute, the way a training loop feeds a layer. The same loop
    # with the whole dx read back (32 MB per step) is reported beside it.
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        dyh = dy.cpu().pin_memory()
        NB = 3  # triple-buffered: step i+1's H2D never waits on step i-1's D2H
        dxh = [torch.empty_like(xh).pin_memory() for _ in range(NB)]
        sumh = torch.empty(NB, dtype=torch.float32).pin_memory()
        xd = [torch.empty_like(x) for _ in range(NB)]
        dyd = [torch.empty_like(dy) for _ in range(NB)]
        dxd = [torch.empty_like(dx) for _ in range(NB)]
        sumd = torch.empty(NB, dtype=torch.float32, device="cuda")
        comp = torch.cuda.current_stream()
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ev_x = [torch.cuda.Event() for _ in range(NB)]
        ev_dy = [torch.cuda.Event() for _ in range(NB)]
        ev_done = [torch.cuda.Event() for _ in range(NB)]
        ev_free = [torch.cuda.Event() for _ in range(NB)]
        for i in range(NB):
            ev_free[i].record(comp)

        def e2e_steps(n, full_dx):
            for i in range(n):
                b = i % NB
                with torch.cuda.stream(s_in):
                    s_in.wait_event(ev_free[b])       # step i-NB no longer uses set b
                    xd[b].copy_(xh, non_blocking=True)
                    ev_x[b].record(s_in)
                    dyd[b].copy_(dyh, non_blocking=True)
                    ev_dy[b].record(s_in)
                comp.wait_event(ev_x[b])              # forward needs x only
                layer.forward(xd[b], y)
                comp.wait_event(ev_dy[b])
                layer.backward(dyd[b], dxd[b])
                if not full_dx:
                    torch.sum(dxd[b], dim=(0, 1), dtype=torch.float32, out=sumd[b])
                ev_done[b].record(comp)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev_done[b])
                    if full_dx:
                        dxh[b].copy_(dxd[b], non_blocking=True)
                    else:
                        sumh[b:b + 1].copy_(sumd[b:b + 1], non_blocking=True)
                    ev_free[b].record(s_out)        # result read out, inputs consumed
            comp.wait_stream(s_out)

        def e2e_ms(full_dx):
            ke = max(1, min(args.steps, 50))
            e2e_steps(NB, full_dx)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            s.record()
            e2e_steps(ke, full_dx)
            e.record()
            torch.cuda.synchronize()
            t = torch.tensor([s.elapsed_time(e) / ke], device="cuda", dtype=torch.float64)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())

        ems = e2e_ms(False)
        ems_full = e2e_ms(True)
        e2e = {"value": world * T / (ems * 1e-3), "unit": "tokens/s",
               "h2d_bytes_per_step": 2 * x.numel() * x.element_size(),
               "d2h_bytes_per_step": 4, "ms_per_step": ems,
               "api": "paper_2501_10714_b200.layer.MoELayer forward+backward (libfsmoe.so C ABI)",
               "copies": "pinned host x and dy in, an fp32 checksum of dx out, on copy streams "
                         "triple-buffered against compute, all inside the timed region",
               "with_full_dx_readback": {"value": world * T / (ems_full * 1e-3), "ms_per_step": ems_full,
                                         "d2h_bytes_per_step": dx.numel() * dx.element_size()}}

    timeline = None
    if args.trace or world > 1:
        # measured per-phase timeline (3 extra steps, outside the timed
        # region): with EP it carries the exposed AlltoAll
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
        if world > 1:
            # every rank's exchange waits: a rank that waits long is waiting for
            # a slower rank (expert load imbalance under capacity), the rank
            # that waits least is on the critical path and its waits are the
            # exchange latency the step really exposes
            per = [None] * world
            dist.all_gather_object(per, timeline["comm_exposed_ms_per_step"])
            timeline["comm_wait_ms_per_step_by_rank"] = per
            timeline["comm_exposed_ms_per_step"] = max(per)
            timeline["exposed_alltoall_ms_per_step"] = min(per)
            timeline["note"] = ("traced run synchronises per phase call; shares, not absolute step "
                                "time. exposed_alltoall = the critical-path rank's exchange waits; "
                                "larger waits on other ranks are expert-load imbalance")

    roof, gflops, gms = gemm_roofline(layer, peaks)
    roof["peak_source"] = peak_kind
    traffic_file = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(traffic_file):
        with open(traffic_file) as f:
            roof["traffic"] = json.load(f).get("bytes_per_step")
    # step roofline (north star): max(GEMM flops at peak, AlltoAll bytes at NVLink)
    C = layer.capacity
    a2a_bytes = 4 * E * C * M * 2 * (world - 1) / world
    t_gemm = gflops / (peaks.get("bf16_tflops", 1590.0) * 1e12) * 1e3
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
    step_roof = {"gemm_flops": gflops, "a2a_bytes_out_per_gpu": a2a_bytes,
                 "a2a_measured": a2a_meas,
                 "roofline_ms": max(t_gemm, t_a2a), "measured_ms": ms,
                 "frac": max(t_gemm, t_a2a) / ms, "gemm_share_of_step": gms / ms,
                 # also against the sustained (power-limited, 4 s back
                 # to back) cuBLAS figure and the 2.25 PFLOP/s spec
                 "frac_vs_sustained": max(gflops / (peaks.get("bf16_tflops_sustained", 1400.0) * 1e12) * 1e3,
                                          t_a2a) / ms,
                 "frac_vs_spec": max(gflops / 2.25e15 * 1e3, t_a2a) / ms,
                 "roofline_tokens_per_s": world * T / (max(t_gemm, t_a2a) * 1e-3)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        xs, wg, wn = cpu_inputs(1024 * (os.cpu_count() or 1), M, E)
        thr = os.cpu_count() or 1
        rate, kind, thr, calls, wall = cpu_reference_rate(args.cpu_seconds, thr, 1024, xs, wg, wn, E,
                                                          -(-1024 * WORKLOAD["top_k"] // E))
        cpu = {"value": rate, "unit": "tokens/s", "cores": thr, "kind": kind,
               "sample": f"{calls} calls x 1024 tokens (d_model {M}, {E} experts, top-{WORKLOAD['top_k']}) of "
                         f"run_gate->dispatch_tokens->combine_tokens over {wall:.1f} s on {thr} "
                         "threads; the reference has no FFN/backward"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random tokens, random-init experts)",
            "config": dict(WORKLOAD, parallelism=f"ep{world}", r_fwd=args.r_fwd, r_bwd=args.r_bwd,
                           capacity=C, **({"gate": gate} if args.gate else {})),
            "clocks": clk, "e2e": e2e, "gpu_launches": launches,
            "roofline": roof, "step_roofline": step_roof, "cpu_baseline": cpu,
        }
        if timeline:
            line["timeline"] = timeline
        print(json.dumps(line), flush=True)
    layer.close()
    if ep:
        ep.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--r-fwd", type=int, default=1)
    ap.add_argument("--r-bwd", type=int, default=1)
    ap.add_argument("--nccl-ctas", type=int, default=16)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--trace", default="", help="write per-rank measured timelines to PATH.rankN.json")
    ap.add_argument("--config", default="gpt2m", choices=sorted(WORKLOADS),
                    help="gpt2m = BASELINE configs[1] (the headline); mixtral = configs[2]; "
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
