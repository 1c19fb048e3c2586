"""The multi-layer backward with both windows of the gradient-partition plan
(model.py; grad_partition.cpp:57-93 step 1 fills the dense window first,
then the MoE window; schedule_sim.cpp:383-434 pre_sync tasks beside the
dense backward) on ONE GPU through the single-GPU multi-rank harness: P
logical ranks, each with its own MoE layers and dense blocks. Every dense
gradient must be summed over the ranks exactly once — in a later layer's
dense window, its MoE window or the tail — so the plan's placement gives the
same pool, outputs and input gradients (bit for bit: the local group sums in
rank order) as syncing everything after the backward."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4])
def test_stack_dense_and_moe_windows_local(world):
    from test_autotune import _samples

    from paper_2501_10714_b200 import plan as P
    from paper_2501_10714_b200.layer import EpGroup, MoEConfig, run_ranks
    from paper_2501_10714_b200.model import MoEStack

    cfg = MoEConfig(tokens=512, model_dim=256, ffn_dim=256, experts=4 * world, top_k=2,
                    gate="sigmoid_topk")
    prof = P.fit_profile(_samples(2e-6))[0]  # comm expensive enough that the plan uses windows
    res = {}
    for sync in ("plan", "tail"):
        groups = EpGroup.local_group(world, torch.cuda.current_device())
        stacks = run_ranks(world, lambda r: MoEStack(cfg, 3, groups[r], plan_profile=prof, sync=sync,
                                                     dense=True, t_olp_dense_ms=0.1))

        def step(r):
            st = stacks[r]
            g = torch.Generator(device="cuda").manual_seed(11 + r)
            x = torch.randn(cfg.tokens, cfg.model_dim, device="cuda", generator=g).to(torch.bfloat16)
            dy = torch.randn(cfg.tokens, cfg.model_dim, device="cuda", generator=g).to(torch.bfloat16)
            y = st.forward(x)
            dx = st.backward(dy)
            return (y.clone(), dx.clone(), st.pool.clone(), list(st.loads), list(st.dense_loads), st.tail)

        res[sync] = run_ranks(world, step)
        run_ranks(world, lambda r: stacks[r].close())
        for gr in groups:
            gr.close()
    plan, tail = res["plan"], res["tail"]
    moe_loads, dense_loads, t = plan[0][3], plan[0][4], plan[0][5]
    n_grad = 4 * cfg.model_dim * cfg.model_dim
    assert sum(dense_loads) > 0, (moe_loads, dense_loads)  # the dense windows were used
    assert sum(moe_loads) + sum(dense_loads) + t == 3 * n_grad
    for r in range(world):
        assert torch.equal(plan[r][0], tail[r][0]), f"rank {r}: y differs"
        assert torch.equal(plan[r][1], tail[r][1]), f"rank {r}: dx differs"
        assert torch.equal(plan[r][2], tail[r][2]), f"rank {r}: synced dense gradients differ"
        assert torch.equal(plan[r][2], plan[0][2])  # replicated: same on every rank
    assert float(plan[0][2].abs().max()) > 0
