"""The glibc libm restatement the gate runs on the device
(paper_2501_10714_b200/csrc/glibc_libm.cuh) against the live libm of this
host, bit for bit, on the CPU: the same source compiled by g++ (no FP
contraction) over millions of arguments — the gate's u1 / 2 pi u2 domains,
the near-1 log window, every cos reduction branch, logits-scale and full-range
exp / log1p arguments, random bit patterns and edge values — plus the
composed normal draw and softplus exactly as proj/src/workload.cpp:90-101.

The reference's noise and softmax / sigmoid weights are only as exact as
these (not correctly rounded) routines; the device restatement is what
makes the noisy gate's indices and weights bit-identical rather than
"within 1e-12".
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "glibc_libm_check")
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-builtin",
                    "-I", os.path.join(ROOT, "paper_2501_10714_b200", "csrc"),
                    os.path.join(ROOT, "tests", "native", "glibc_libm_check.cpp"), "-o", exe, "-lm"],
                   check=True)
    return exe


def test_generated_tables_match_this_libm():
    """glibc_libm_data.h is what tools/extract_glibc_libm.py reads out of this
    host's libm (the sha256 the addresses belong to)."""
    import hashlib
    import importlib.util
    spec = importlib.util.spec_from_file_location("ex", os.path.join(ROOT, "tools", "extract_glibc_libm.py"))
    ex = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ex)
    if hashlib.sha256(open(ex.LIBM, "rb").read()).hexdigest() != ex.SHA256:
        pytest.skip("a different libm build (the restatement pins glibc 2.39's)")
    import struct
    data = open(ex.LIBM, "rb").read()
    hdr = open(ex.OUT).read()
    for name, addr in ex.SCALARS:
        (w,) = struct.unpack_from("<Q", data, addr)
        assert f"{name} = 0x{w:016x}ULL" in hdr, name
    for name, addr, n in ex.TABLES:
        words = struct.unpack_from(f"<{n}Q", data, addr)
        assert f"0x{words[0]:016x}ULL" in hdr and f"0x{words[-1]:016x}ULL" in hdr, name


@pytest.mark.parametrize("seed", [1, 2])
def test_restatement_is_bit_identical_to_host_libm(tmp_path, seed):
    exe = _build(tmp_path)
    out = subprocess.run([exe, "1500000", str(seed)], check=True, capture_output=True, text=True).stdout
    rows = {ln.split()[0]: (int(ln.split()[1]), int(ln.split()[2]), ln.split()[3])
            for ln in out.strip().splitlines()}
    assert set(rows) == {"log", "exp", "log1p", "cos", "normal", "softplus"}
    for name, (n, bad, first) in rows.items():
        assert n >= 1500000, name
        assert bad == 0, f"{name}: {bad} of {n} differ from the host libm (first at {first})"
