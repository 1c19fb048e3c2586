"""Host side of the on-box planning loop (paper_2501_10714_b200/autotune.py):
the bench CSV in the reference's format (json_io.cpp:262-300) and
fit_profile -> plan_layer on synthetic alpha-beta samples (CPU)."""
import pytest

from paper_2501_10714_b200 import autotune
from paper_2501_10714_b200.layer import MoEConfig


def _samples(a2a_beta):
    out = []
    for k, a, b in (("a2a", 0.02, a2a_beta), ("ag", 0.02, 1e-7), ("rs", 0.02, 1e-7),
                    ("ar", 0.03, 2e-7), ("gemm", 0.005, 2.5e-11)):
        for n in (1e6, 2e6, 4e6, 8e6) if k != "gemm" else (1e9, 2e9, 4e9, 8e9):
            out.append((k, n, a + b * n))
    return out


def test_bench_csv_round_trip_and_reference_errors():
    s = _samples(1e-7)
    text = autotune.write_bench_csv(s)
    assert text.splitlines()[0] == "kind,n,t_ms"
    assert autotune.read_bench_csv(text) == [(k, float(n), float(t)) for k, n, t in s]
    with pytest.raises(ValueError, match="expected header kind,n,t_ms"):
        autotune.read_bench_csv("k,n,t\n")
    with pytest.raises(ValueError, match="unknown kind 'xx'"):
        autotune.read_bench_csv("kind,n,t_ms\nxx,1,2\n")
    with pytest.raises(ValueError, match="expected 3 fields, got 2"):
        autotune.read_bench_csv("kind,n,t_ms\na2a,1\n")


def test_plan_reacts_to_comm_cost():
    cfg = MoEConfig(tokens=16384, model_dim=1024, ffn_dim=4096, experts=16, top_k=1)
    cheap = autotune.plan(cfg, _samples(1e-9), world=4)
    dear = autotune.plan(cfg, _samples(2e-6), world=4)
    assert cheap["min_r2"] > 0.999 and dear["min_r2"] > 0.999
    for p in (cheap, dear):
        assert 1 <= p["r_fwd"] <= 8 and 1 <= p["r_bwd"] <= 8
    # expensive AlltoAll relative to the GEMM -> more pipelining
    assert dear["t_moe_fwd_ms"] > cheap["t_moe_fwd_ms"]
    assert dear["r_fwd"] >= cheap["r_fwd"]
