"""Close the FSMoE planning loop on this box:
profile -> bench CSV -> fit_profile -> plan_layer, then validate the chosen
pipeline degrees against the measured step time of every r in 1..R for both
EP transports (NCCL grouped send/recv, where chunking is the overlap
mechanism, and the fused peer-memory transport).

    torchrun --nproc-per-node N tools/plan_on_box.py [--out gpurun_out/plan]
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def step_ms(layer, x, dy, steps=20, warmup=3):
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    for _ in range(warmup):
        layer.forward(x, y)
        layer.backward(dy, dx)
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        layer.forward(x, y)
        layer.backward(dy, dx)
    e.record()
    torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e) / steps], device="cuda", dtype=torch.float64)
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/plan")
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--model-dim", type=int, default=1024)
    ap.add_argument("--ffn-dim", type=int, default=4096)
    ap.add_argument("--experts", type=int, default=16)
    ap.add_argument("--top-k", type=int, default=1)
    ap.add_argument("--r-max", type=int, default=4)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2501_10714_b200 import autotune
    from paper_2501_10714_b200.layer import EpGroup, MoEConfig, MoELayer

    cfg = MoEConfig(tokens=args.tokens, model_dim=args.model_dim, ffn_dim=args.ffn_dim,
                    experts=args.experts, top_k=args.top_k, gate="noisy_topk", ffn="simple")
    samples, vol = autotune.collect(cfg, world)
    p = autotune.plan(cfg, samples, world, r_max=args.r_max)
    os.makedirs(args.out, exist_ok=True)
    if rank == 0:
        autotune.write_bench_csv(samples, os.path.join(args.out, f"bench_p{world}.csv"))

    g = torch.Generator(device="cuda").manual_seed(5 + rank)
    x = torch.randn(cfg.tokens, cfg.model_dim, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(cfg.tokens, cfg.model_dim, device="cuda", generator=g).to(torch.bfloat16)
    measured = {}
    for transport in ("nccl", "peer"):
        if world == 1 and transport == "nccl":
            continue
        os.environ["FSMOE_EP_TRANSPORT"] = transport
        ep = EpGroup(world, rank, local, max_ctas=16) if world > 1 else None
        rows = {}
        for r in range(1, args.r_max + 1):
            cfg.r_fwd = cfg.r_bwd = r
            layer = MoELayer(cfg, ep, init_seed=1)
            rows[r] = step_ms(layer, x, dy)
            layer.close()
        cfg.r_fwd, cfg.r_bwd = p["r_fwd"], p["r_bwd"]
        layer = MoELayer(cfg, ep, init_seed=1)
        rows["planned"] = step_ms(layer, x, dy)
        layer.close()
        if ep:
            ep.close()
        measured[transport] = rows
    if rank == 0:
        rep = {"world": world, "layer": {"tokens": cfg.tokens, "model_dim": cfg.model_dim,
                                         "ffn_dim": cfg.ffn_dim, "experts": cfg.experts,
                                         "top_k": cfg.top_k},
               "samples": samples, "plan": p, "measured_step_ms": measured,
               "best_r": {t: min((k for k in v if k != "planned"), key=lambda k: v[k])
                          for t, v in measured.items()}}
        with open(os.path.join(args.out, f"plan_p{world}.json"), "w") as f:
            json.dump(rep, f, indent=1)
        print(json.dumps({"plan": {k: p[k] for k in ("r_fwd", "r_bwd", "t_moe_fwd_ms", "t_moe_bwd_ms")},
                          "measured": measured, "best_r": rep["best_r"]}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
