"""Measure the gradient-partition plan on this box: an
L-layer MoE stack (BASELINE configs[1] layers) whose dense blocks each hand
back a 4*M^2 fp32 gradient; forward + backward step time with the plan's
slot placement vs one allreduce of the whole pool after the backward vs no
dense gradient at all.

    torchrun --nproc-per-node N tools/stack_on_box.py [--layers 4] [--out gpurun_out/stack]
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--steps", type=int, default=10)
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

    cfg = MoEConfig(tokens=16384, model_dim=1024, ffn_dim=4096, experts=16, top_k=1)
    samples, _ = autotune.collect(cfg, world)
    prof = P.fit_profile(samples)[0]
    ep = EpGroup(world, rank, local, max_ctas=16)
    g = torch.Generator(device="cuda").manual_seed(7 + rank)
    x = torch.randn(cfg.tokens, cfg.model_dim, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(cfg.tokens, cfg.model_dim, device="cuda", generator=g).to(torch.bfloat16)
    res = {}
    for name, sync, ng in (("no_dense_grad", "tail", 0), ("tail", "tail", None), ("plan", "plan", None)):
        st = MoEStack(cfg, args.layers, ep, n_grad=ng, plan_profile=prof, sync=sync)
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
        res[name] = {"step_ms": float(t.item()), "slot_loads": list(st.loads), "tail": st.tail,
                     "n_grad": st.n_grad}
        if name == "plan":
            res[name]["plan"] = {"layers": st.plan_layers, "tail": st.plan_tail}
        st.close()
    ep.close()
    if rank == 0:
        os.makedirs(args.out, exist_ok=True)
        rep = {"world": world, "layers": args.layers, "config": "BASELINE configs[1] layer x L, "
               "dense gradient 4*M^2 fp32 per layer", "results": res}
        with open(os.path.join(args.out, f"stack_p{world}.json"), "w") as f:
            json.dump(rep, f, indent=1)
        print(json.dumps({k: {kk: v[kk] for kk in ("step_ms", "slot_loads", "tail")}
                          for k, v in res.items()}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
