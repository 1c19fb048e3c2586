"""Host logic of the multi-layer gradient-partition executor (model.py):
rounding the plan's real-valued window loads to integer slices must conserve
every element, respect availability (position i only syncs gradient produced
at positions < i) and keep the tail non-negative — for the MoE windows
(n_first_moe + x_g) and the dense windows (n_first_dense) together, on plans
the bit-exact planner port produces (grad_partition.cpp:185-228)."""
import numpy as np
import pytest

from paper_2501_10714_b200 import plan as P
from paper_2501_10714_b200.model import _parse_plan, slot_loads


def _samples(a2a_beta):
    out = []
    for k, a, b in (("a2a", 0.02, a2a_beta), ("ag", 0.02, 1e-7), ("rs", 0.02, 1e-7),
                    ("ar", 0.03, 2e-7), ("gemm", 0.005, 2.5e-11)):
        for n in (1e6, 2e6, 4e6, 8e6) if k != "gemm" else (1e9, 2e9, 4e9, 8e9):
            out.append((k, n, a + b * n))
    return out


@pytest.mark.parametrize("t_dense,a2a_beta,L", [(0.0, 2e-6, 3), (0.1, 2e-6, 3), (0.5, 1e-7, 5),
                                                 (2.0, 2e-6, 8)])
def test_slot_loads_conserve_and_respect_availability(t_dense, a2a_beta, L):
    prof = P.fit_profile(_samples(a2a_beta))[0]
    layer = P.Layer(batch=1, heads=1, seq_len=4096, model_dim=1024, hidden_scale=4, capacity_factor=1.0,
                    ffn="simple", experts=8, top_k=2)
    vol = P.derive_volumes(layer, (4, 4, 1, 1, 4, 1))
    n_grad = 4 * 1024 * 1024
    out = P.build_partition_plan([(vol, t_dense, float(n_grad))] * L, prof, (0, 60, 0.8, 0.9, 3))
    layers, tail_plan = _parse_plan(out, L)
    moe, dense, tail = slot_loads(layers, n_grad, L)
    assert all(v >= 0 for v in moe + dense) and tail >= 0
    assert sum(moe) + sum(dense) + tail == L * n_grad
    cum = 0
    for i in range(L):
        cum += dense[i]
        assert cum <= i * n_grad  # dense window: gradient of earlier positions only
        cum += moe[i]
        assert cum <= (i + 1) * n_grad  # MoE window: its own position's too
    if t_dense == 0.0:
        assert sum(dense) == 0
    # the integer loads follow the plan's real-valued ones to within rounding
    plan_total = sum(a["n_first"] + a["x_g"] for a in layers)
    assert abs(sum(moe) + sum(dense) - plan_total) <= L
    assert abs(tail - tail_plan["tail_elements"]) <= L
