"""The reference's OWN unit suites run against this repo's drop-in.

oracle/Makefile `reftests` compiles /root/reference/proj/tests/test_*.cpp
unchanged — with a doctest stand-in (oracle/doctest_shim/doctest.h, the
framework is absent from the image) — against include/fsmoe/*.hpp and
libfsmoe.so instead of the reference library. The binaries land in
oracle/_ref/tests/ (git-ignored, built by __graft_entry__.build() where the
reference exists, and shipped to the GPU box with the tree).

* test_workload — run_gate / dispatch_tokens / combine_tokens on host
  Matrix values (the C++ entry points the reference's callers use,
  test_workload.cpp:160-512): every gating KAT and brute-force oracle of the
  reference, executed by the B200 kernels behind the drop-in (GPU).
* test_cost_models / test_schedule_sim / test_pipeline_optimizer /
  test_grad_partition — the planner KATs (host code, CPU).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "tests")


def _run(name):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make -C oracle reftests needs /root/reference)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    summary = [ln for ln in r.stdout.splitlines() if ln.startswith("[doctest-shim]")]
    assert summary and "| 0 failed | assertions:" in summary[-1] and summary[-1].endswith("| 0 failed"), tail
    return summary[-1]


@pytest.mark.parametrize("name", ["test_cost_models", "test_schedule_sim", "test_pipeline_optimizer",
                                  "test_grad_partition"])
def test_reference_planner_suite(name):
    _run(name)


@pytest.mark.gpu
def test_reference_workload_suite_on_gpu():
    """The reference's routing KATs through fsmoe::run_gate / dispatch_tokens /
    combine_tokens (libfsmoe.so -> libfsmoe_cuda.so)."""
    out = _run("test_workload")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "reference_test_workload.txt"), "w") as f:
        f.write(out + "\n")
