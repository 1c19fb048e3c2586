"""bench.py host logic on CPU: the trace timeline summary (exposed comm time),
the nvidia-smi clock sampler's parsing and the workload table the JSON
contract names."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_timeline_summary_exposed_comm():
    # comm [0, 10) us and [20, 30) us; compute covers [5, 25) us -> exposed 5 + 5
    ev = [{"name": "fwd.dispatch", "tid": 0, "ts": 0.0, "dur": 10.0},
          {"name": "fwd.combine", "tid": 0, "ts": 20.0, "dur": 10.0},
          {"name": "fwd.expert[0]", "tid": 2, "ts": 5.0, "dur": 20.0}]
    out = bench.timeline_summary(json.dumps({"traceEvents": ev}), steps=1)
    assert out["comm_exposed_ms_per_step"] == pytest.approx(0.010)
    assert out["comm_ms_per_step"] == pytest.approx(0.020)
    assert out["phase_ms_per_step"]["fwd.expert"] == pytest.approx(0.020)
    assert out["traced_ms_per_step"] == pytest.approx(0.030)


def test_clock_sampler_parses_region_samples(tmp_path):
    s = bench.ClockSampler(0)
    s.path = str(tmp_path / "clk.csv")
    rows = [
        "0, 1965, 1965, 200.0, 0x0000000000000001, Not Active, Not Active, Not Active, Not Active",  # idle, before
        "0, 1800, 1965, 990.0, 0x0000000000000004, Not Active, Not Active, Not Active, Active",
        "0, 1700, 1965, 995.0, 0x0000000000000014, Not Active, Not Active, Not Active, Active",
        "0, 1965, 1965, 700.0, 0x0000000000000000, Not Active, Not Active, Not Active, Not Active",
    ]
    with open(s.path, "w") as f:
        f.write("\n".join(rows) + "\n")
    s.n0 = 1  # the first line was written before the timed region

    class Done:  # stands in for the finished nvidia-smi process
        def terminate(self):
            pass

        def wait(self, timeout=None):
            return 0

    s.proc = Done()
    out = s.stop()
    assert out["samples"] == 3
    assert out["sm_mhz"] == 1800.0
    assert out["sm_max_mhz"] == 1965.0
    assert out["reasons"] == ["sw_power_cap", "sync_boost"]


def test_workloads_table():
    assert bench.WORKLOADS["gpt2m"]["tokens_per_gpu"] == 16384
    assert bench.WORKLOADS["mixtral"]["d_ffn"] == 14336
    assert set(bench.GATES) == {"noisy_topk", "sigmoid_topk", "cosine_topk", "expert_choice"}
    for w in bench.WORKLOADS.values():
        assert {"workload", "tokens_per_gpu", "d_model", "d_ffn", "experts", "top_k"} <= set(w)


def test_reference_pass_routes_the_gpu_arms_instance():
    """The reference arm and cpu_baseline route the GPU arm's instance: same
    T, capacity_tokens(k, f) (workload.cpp:43-51), all threads on the whole
    instance (a tiny shape here)."""
    assert bench.WORKLOADS["mixtral"] is bench.WORKLOAD  # the headline default
    old = bench.WORKLOAD
    try:
        bench.WORKLOAD = dict(old, tokens_per_gpu=256, d_model=64, experts=8, top_k=2)
        assert bench.instance_capacity() == 64
        x, wg, wn = bench.cpu_inputs(256, 64, 8)
        rate, kind, thr, wall = bench.cpu_reference_pass(2, x, wg, wn, 8, 2, 64)
        assert thr == 2 and rate > 0 and wall > 0 and kind in ("reference", "port")
    finally:
        bench.WORKLOAD = old
    assert bench.cpu_threads_for(32768, 4096, 8, 8192) >= 1


def test_cpu_layer_restatement_small():
    """The labelled CPU restatement of the expert FFN fwd+bwd runs and reports
    a positive rate (tiny shape here; the bench uses the workload's)."""
    rate, secs = bench.cpu_layer_restatement(64, 128, True, 2, 2, tokens=16)
    assert rate > 0 and secs > 0
    rate, secs = bench.cpu_layer_restatement(64, 128, False, 1, 2, tokens=16)
    assert rate > 0 and secs > 0


def test_reference_arm_steps_are_bounded(monkeypatch, capsys):
    """--impl reference with many steps: each step routes a sub-instance so the
    whole run stays within the time budget (the reference's cost is linear in
    the tokens); with the default 20 steps the full instance is kept."""
    import argparse
    import numpy as np
    T = bench.WORKLOAD["tokens_per_gpu"]
    seen = []

    def fake_pass(threads, x, wg, wn, E, k, cap):
        seen.append((x.shape[0], cap))
        return threads * x.shape[0] / (9.0 * x.shape[0] / T), "reference", threads, 9.0 * x.shape[0] / T

    monkeypatch.setattr(bench, "cpu_reference_pass", fake_pass)
    monkeypatch.setattr(bench, "cpu_threads_for", lambda *a: 4)
    monkeypatch.setattr(bench, "cpu_inputs", lambda t, M, E: (np.zeros((t, 8)), None, None))
    bench.reference_arm(argparse.Namespace(steps=100, warmup=3, gpus=1))
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    t_s = seen[-1][0]
    assert t_s < T and t_s % 64 == 0 and 100 * 9.0 * t_s / T <= 240.0 + 1e-6
    assert "first" in line["cpu_baseline"]["sample"]
    seen.clear()
    bench.reference_arm(argparse.Namespace(steps=20, warmup=3, gpus=1))
    assert seen[-1][0] == T
