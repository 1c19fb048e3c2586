"""Multi-layer backward executing the gradient-partition plan (model.py,
SURVEY §8f row 2) on >= 2 GPUs: every layer's replicated dense gradient is
allreduced exactly once — inside later layers' MoE slots or in the tail — and
the MoE results do not depend on where the syncs ran."""
import os
import socket
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
        import torch.distributed as dist

        from paper_2501_10714_b200 import plan as P
        from paper_2501_10714_b200.layer import EpGroup, MoEConfig
        from paper_2501_10714_b200.model import MoEStack
        from test_autotune import _samples
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", rank))
        cfg = MoEConfig(tokens=512, model_dim=256, ffn_dim=256, experts=4 * world, top_k=1)
        prof = P.fit_profile(_samples(2e-6))[0]  # expensive comm: the plan uses the slots
        ep = EpGroup(world, rank, rank)
        n_grad = 4096
        out = {}
        for sync in ("plan", "tail"):
            st = MoEStack(cfg, 3, ep, n_grad=n_grad, plan_profile=prof, sync=sync)
            g = torch.Generator(device="cuda").manual_seed(11 + rank)
            x = torch.randn(cfg.tokens, cfg.model_dim, device="cuda", generator=g).to(torch.bfloat16)
            dy = torch.randn(cfg.tokens, cfg.model_dim, device="cuda", generator=g).to(torch.bfloat16)
            y = st.forward(x)
            dx = st.backward(dy, produce=lambda j, seg: seg.fill_(float((rank + 1) * (j + 1))))
            torch.cuda.synchronize()
            exp = torch.cat([torch.full((n_grad,), float((j + 1) * world * (world + 1) // 2),
                                        device="cuda") for j in range(3)])
            out[sync] = (y.clone(), dx.clone(), torch.equal(st.pool, exp), list(st.loads), st.tail)
            st.close()
        ok = (out["plan"][2] and out["tail"][2] and torch.equal(out["plan"][0], out["tail"][0])
              and torch.equal(out["plan"][1], out["tail"][1]) and sum(out["plan"][3]) > 0)
        ep.close()
        dist.destroy_process_group()
        q.put((rank, "ok" if ok else "bad", {"loads": out["plan"][3], "tail": out["plan"][4],
                                             "pool_ok": [out["plan"][2], out["tail"][2]]}))
    except Exception as e:
        import traceback
        q.put((rank, "error " + repr(e) + traceback.format_exc()[-1500:], {}))


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_stack_backward_syncs_every_gradient_once():
    import torch.multiprocessing as mp
    world = min(4, torch.cuda.device_count())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(s == "ok" for _, s, _ in res), res
