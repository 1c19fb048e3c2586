"""SURVEY.md §8d C4 sweep on this box: for each layer shape, profile ->
fit_profile -> plan_layer, the simulator's predicted fwd / bwd makespan for
every r (schedule_sim port), and the measured forward and backward time for
every r on both EP transports. Records planner r vs measured-best r per
point (the paper's "online profiling picks a near-optimal degree" claim).

    torchrun --nproc-per-node N tools/sweep_on_box.py [--out gpurun_out/sweep] [--quick]
"""
import argparse
import itertools
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _max(v):
    if dist.is_initialized():
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return v


def fwd_bwd_ms(layer, x, dy, steps=10, warmup=3):
    """(forward ms, backward ms): forward-only loop, then fwd+bwd loop;
    backward = difference (max over ranks each)."""
    y, dx = torch.empty_like(x), torch.empty_like(x)
    for _ in range(warmup):
        layer.forward(x, y)
        layer.backward(dy, dx)
    out = []
    for with_bwd in (False, True):
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            layer.forward(x, y)
            if with_bwd:
                layer.backward(dy, dx)
        e.record()
        torch.cuda.synchronize()
        out.append(_max(s.elapsed_time(e) / steps))
    return out[0], out[1] - out[0]


def grid(quick, wide=False):
    if quick:
        return [(4096, 1024, 2, 8, 2), (16384, 1024, 4, 16, 1)]
    if wide:  # round 2: the C4 corners round 1 left out (T 64k, E 64, M 4096)
        return list(itertools.product((4096, 16384, 65536), (1024, 4096), (4,), (8, 64), (1, 2)))
    pts = []
    for T, M, hs, E, k in itertools.product((4096, 16384), (1024, 2048), (2, 4), (8, 32), (1, 2)):
        pts.append((T, M, hs, E, k))
    return pts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweep")
    ap.add_argument("--r-max", type=int, default=4)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--wide", action="store_true")
    ap.add_argument("--transports", default="peer,ce")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2501_10714_b200 import autotune
    from paper_2501_10714_b200 import plan as P
    from paper_2501_10714_b200.layer import EpGroup, MoEConfig, MoELayer

    transports = [t for t in args.transports.split(",") if world > 1 or t == "peer"]
    rows = []
    t0 = time.time()
    for (T, M, hs, E, k) in grid(args.quick, args.wide):
        if E % world:
            continue
        cfg = MoEConfig(tokens=T, model_dim=M, ffn_dim=hs * M, experts=E, top_k=k,
                        gate="noisy_topk", ffn="simple")
        samples, vol = autotune.collect(cfg, world, reps=5)
        p = autotune.plan(cfg, samples, world, r_max=args.r_max)
        prof = p["profile"]
        pred = {}
        for r in range(1, args.r_max + 1):
            f = P.simulate_stage(vol, prof, 1, r)
            b = P.simulate_stage(vol, prof, 2, r)
            pred[r] = (float(f[0]), float(b[0]))
        g = torch.Generator(device="cuda").manual_seed(5 + rank)
        x = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
        dy = torch.randn(T, M, device="cuda", generator=g).to(torch.bfloat16)
        meas = {}
        ep = EpGroup(world, rank, local, max_ctas=16) if world > 1 else None
        for tr in transports:
            cfg.transport = tr
            m = {}
            for r in range(1, args.r_max + 1):
                cfg.r_fwd = cfg.r_bwd = r
                layer = MoELayer(cfg, ep, init_seed=1)
                m[r] = fwd_bwd_ms(layer, x, dy)
                layer.close()
            meas[tr] = m
        # FSMoE's online loop as bench.py runs it: the plan refined on the layer
        cfg.transport = ""
        rf, rb, cand = autotune.refine(cfg, ep, (p["r_fwd"], p["r_bwd"]), x, dy, r_max=args.r_max,
                                       steps=5, transports=tuple(transports) if world > 1 else None)
        refined = {"transport": cfg.transport or "peer", "r": rf,
                   "candidates_ms": {str(c): v for c, v in cand.items()}}
        if ep:
            ep.close()
        del x, dy
        torch.cuda.empty_cache()
        row = {"T": T, "M": M, "H": hs * M, "E": E, "k": k, "capacity": int(vol[6]),
               "plan": {"r_fwd": p["r_fwd"], "r_bwd": p["r_bwd"], "case_fwd": p["case_fwd"],
                        "case_bwd": p["case_bwd"], "t_moe_fwd_ms": p["t_moe_fwd_ms"],
                        "t_moe_bwd_ms": p["t_moe_bwd_ms"], "min_r2": p["min_r2"]},
               "predicted_ms": {r: v for r, v in pred.items()},
               "measured_ms": {tr: {r: v for r, v in m.items()} for tr, m in meas.items()},
               "refined": refined}
        step = {(tr, r): v[0] + v[1] for tr, m in meas.items() for r, v in m.items()}
        best = min(step, key=step.get)
        row["best_step"] = {"transport": best[0], "r": best[1], "ms": step[best],
                            "refined_over_best": step[(refined["transport"], refined["r"])] / step[best],
                            "plan_peer_over_best": step[(transports[0], max(p["r_fwd"], p["r_bwd"]))] / step[best]}
        for tr, m in meas.items():
            bf = min(m, key=lambda r: m[r][0])
            bb = min(m, key=lambda r: m[r][1])
            row[f"best_{tr}"] = {"r_fwd": bf, "r_bwd": bb,
                                 "plan_fwd_over_best": m[p["r_fwd"]][0] / m[bf][0],
                                 "plan_bwd_over_best": m[p["r_bwd"]][1] / m[bb][1]}
        rows.append(row)
        if rank == 0:
            print(json.dumps({k_: row[k_] for k_ in ("T", "M", "H", "E", "k", "plan", "best_step")}
                             | {f"best_{tr}": row[f"best_{tr}"] for tr in meas},
                             default=float), flush=True)
    if rank == 0:
        os.makedirs(args.out, exist_ok=True)
        with open(os.path.join(args.out, f"sweep_p{world}.json"), "w") as f:
            json.dump({"world": world, "wall_s": time.time() - t0, "points": rows}, f, indent=1,
                      default=float)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
