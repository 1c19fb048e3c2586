"""The FSMoE planning loop on the B200: on-box profile ->
bench CSV -> fit_profile -> plan_layer (the bit-exact reference planner) ->
online refinement on the real layer (autotune.refine), against the measured
step time at every degree r = 1..4. Runs on one GPU (collectives degenerate
to local copies there, so the plan is about GEMM chunking and wave
quantisation); the measured table is written for profiles/."""
import json
import os

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("shape", [dict(tokens=16384, model_dim=1024, ffn_dim=4096, experts=16, top_k=1),
                                   dict(tokens=4096, model_dim=1600, ffn_dim=6400, experts=8, top_k=2)])
def test_profile_fit_plan_refine(shape):
    from paper_2501_10714_b200 import autotune
    from paper_2501_10714_b200.layer import MoEConfig, MoELayer
    cfg = MoEConfig(gate="noisy_topk", ffn="simple", **shape)
    samples, vol = autotune.collect(cfg, 1, r_max=4)
    text = autotune.write_bench_csv(samples)
    assert autotune.read_bench_csv(text) == [(k, float(n), float(t)) for k, n, t in samples]
    p = autotune.plan(cfg, samples, 1, r_max=4)
    assert 1 <= p["r_fwd"] <= 4 and 1 <= p["r_bwd"] <= 4
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(cfg.tokens, cfg.model_dim, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(cfg.tokens, cfg.model_dim, device="cuda", generator=g).to(torch.bfloat16)
    measured = {}
    for r in range(1, 5):
        cfg.r_fwd = cfg.r_bwd = r
        layer = MoELayer(cfg, init_seed=1)
        measured[r] = autotune.step_ms(layer, x, dy)
        layer.close()
    rf, rb, cand = autotune.refine(cfg, None, (p["r_fwd"], p["r_bwd"]), x, dy, r_max=4)
    best = min(measured, key=measured.get)
    # the refined choice is the fastest of its candidates, and within 5 % of
    # the fastest degree overall (timing noise between the two measurements)
    assert cand[rf] == min(cand.values())
    assert measured[rf] <= 1.05 * measured[best], (rf, measured)
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, f"planner_loop_T{cfg.tokens}_M{cfg.model_dim}.json"), "w") as f:
            json.dump({"shape": shape, "plan": {k: p[k] for k in ("r_fwd", "r_bwd")},
                       "profile": p["profile"], "min_r2": p["min_r2"], "measured_step_ms": measured,
                       "refined": [rf, rb], "refine_candidates_ms": cand, "best_r": best,
                       "planned_over_best": measured[max(p["r_fwd"], p["r_bwd"])] / measured[best]}, f, indent=1)
