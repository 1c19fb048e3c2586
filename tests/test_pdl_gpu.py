"""Programmatic dependent launch changes scheduling only: a layer step (gate,
routing, permutations, expert GEMMs, gate backward) run with it on (the
default) and off (FSMOE_PDL=0, read once per process, so each in its own
process) gives bitwise-identical outputs and gradients."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r})
from paper_2501_10714_b200.layer import MoEConfig, MoELayer
cfg = MoEConfig(tokens=4096, model_dim=1024, ffn_dim=1792, experts=8, top_k=2, gate="noisy_topk",
                ffn="gated3", precision="bf16", seed=3)
layer = MoELayer(cfg, init_seed=4)
g = torch.Generator(device="cuda").manual_seed(8)
x = torch.randn(4096, 1024, device="cuda", generator=g).to(torch.bfloat16)
dy = torch.randn(4096, 1024, device="cuda", generator=g).to(torch.bfloat16)
outs = []
for _ in range(2):  # a second step reuses every buffer
    y = layer.forward(x)
    dx = layer.backward(dy)
    torch.cuda.synchronize()
    outs.append({{"y": y.cpu(), "dx": dx.cpu(), "g_w1": layer.g_w1.cpu(), "g_w2": layer.g_w2.cpu(),
                  "g_gate": layer.g_gate.cpu(), "g_noise": layer.g_noise.cpu()}})
torch.save(outs, sys.argv[1])
"""


def _run(tmp_path, pdl):
    out = str(tmp_path / f"pdl{pdl}.pt")
    env = dict(os.environ, FSMOE_PDL=str(pdl))
    subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), out], env=env, check=True, timeout=600)
    return torch.load(out)


def test_pdl_on_off_bitwise(tmp_path):
    on, off = _run(tmp_path, 1), _run(tmp_path, 0)
    for step_on, step_off in zip(on, off):
        for k in step_on:
            assert torch.equal(step_on[k], step_off[k]), k
