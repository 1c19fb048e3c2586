"""Measure the gradient-partition plan on this box (SURVEY §8f row 2 and
BASELINE configs[4]: the other routing functions at the GPT-2-XL shape with
adaptive gradient partitioning enabled): an L-layer stack of dense block +
MoE layer (model.MoEStack, dense=True: each dense block hands back a 4 M^2
fp32 gradient and its backward is the plan's dense window), forward +
backward step time with the plan's placement (dense windows + MoE windows +
tail) vs one allreduce of the whole pool after the backward vs no gradient
sync at all (the lower bound).

    torchrun --nproc-per-node N tools/stack_on_box.py [--config gpt2xl --gate G] [--layers 4]
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {
    "gpt2m": dict(tokens=16384, model_dim=1024, ffn_dim=4096, experts=16, top_k=1),
    "gpt2xl": dict(tokens=4096, model_dim=1600, ffn_dim=6400, experts=8, top_k=2),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--config", default="gpt2xl", choices=sorted(SHAPES))
    ap.add_argument("--gate", default="noisy_topk")
    ap.add_argument("--out", default="gpurun_out/stack")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2501_10714_b200 import autotune
    from paper_2501_10714_b200 import plan as P
    from paper_2501_10714_b200.layer import EpGroup, MoEConfig
    from paper_2501_10714_b200.model import MoEStack

    sh = SHAPES[args.config]
    cfg = MoEConfig(gate=args.gate, proj_dim=64 if args.gate == "cosine_topk" else 0, **sh)
    samples, _ = autotune.collect(cfg, world)
    prof = P.fit_profile(samples)[0]
    ep = EpGroup(world, rank, local, max_ctas=16)
    g = torch.Generator(device="cuda").manual_seed(7 + rank)
    x = torch.randn(cfg.tokens, cfg.model_dim, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(cfg.tokens, cfg.model_dim, device="cuda", generator=g).to(torch.bfloat16)
    res = {}
    t_dense = None
    for name in ("none", "tail", "plan"):
        st = MoEStack(cfg, args.layers, ep, plan_profile=prof, sync=name, dense=True, t_olp_dense_ms=t_dense)
        t_dense = st.t_olp_dense_ms  # measured once, the same window for every placement

        def step():
            st.forward(x)
            st.backward(dy)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.steps):
            step()
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / args.steps], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name] = {"step_ms": float(t.item()), "moe_window_loads": list(st.loads),
                     "dense_window_loads": list(st.dense_loads), "tail": st.tail, "n_grad": st.n_grad,
                     "tokens_per_s": world * cfg.tokens / (float(t.item()) * 1e-3)}
        if name == "plan":
            res[name]["plan"] = {"layers": st.plan_layers, "tail": st.plan_tail,
                                 "t_olp_dense_ms": st.t_olp_dense_ms}
        st.close()
    ep.close()
    if rank == 0:
        os.makedirs(args.out, exist_ok=True)
        rep = {"world": world, "layers": args.layers, "gate": args.gate,
               "config": f"{args.config} MoE layer x L, each behind a dense block with a 4*M^2 fp32 "
                         "gradient (adaptive gradient partitioning: dense + MoE windows + tail)",
               "shape": sh, "results": res}
        with open(os.path.join(args.out, f"stack_{args.config}_{args.gate}_p{world}.json"), "w") as f:
            json.dump(rep, f, indent=1)
        print(json.dumps({k: {kk: v[kk] for kk in ("step_ms", "moe_window_loads", "dense_window_loads", "tail")}
                          for k, v in res.items()}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
