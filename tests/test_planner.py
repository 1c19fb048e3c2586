"""Host control plane (libfsmoe.so: cost models, schedule simulator, pipeline
optimizer, gradient partitioner, capacity/volumes) vs the REFERENCE compiled
from /root/reference (oracle/_ref) — bit-identical outputs on randomized
instances — and the reference test suites' known-answer tests
(proj/tests/test_pipeline_optimizer.cpp, test_schedule_sim.cpp,
test_grad_partition.cpp, test_workload.cpp). CPU only."""
import numpy as np
import pytest

from paper_2501_10714_b200 import plan
from paper_2501_10714_b200._native import ConfigError

pyoracle = pytest.importorskip("pyoracle")
needs_ref = pytest.mark.skipif(not pyoracle.available("reference"),
                               reason="reference oracle not built (make -C oracle ref)")


def ref():
    return pyoracle.RefPlanner()


def prof(a2a, ag, rs, ar, gemm):
    return np.array([*a2a, *ag, *rs, *ar, *gemm], dtype=float)


REF_PROFILE = prof((1.0, 1e-6), (0.1, 1e-6), (0.1, 1e-6), (1.0, 1e-6), (0.25, 1e-9))
REF_VOL = np.array([8e6, 2e6, 2e6, 8e9, 2, 0, 0], dtype=float)


# ------------------------------------------------------------------ KATs --

def test_capacity_and_volumes_kats():
    # test_workload.cpp:58-132
    L = plan.Layer(batch=4, heads=16, seq_len=1024, model_dim=1024, hidden_scale=2,
                   capacity_factor=1.2, experts=8, top_k=2)
    assert plan.capacity_tokens(L) == 1229
    assert plan.capacity_tokens(plan.Layer(2, 16, 4, 1024, 2, 1.0, False, "simple", 8, 1)) == 1
    assert plan.capacity_tokens(plan.Layer(1, 16, 8, 1024, 2, 1.2, True, "simple", 8, 2)) == 16
    v = plan.derive_volumes(L, (32, 8, 2, 4, 8, 4))
    assert list(v) == [2516992.0, 1258496.0, 1258496.0, 2577399808.0, 2.0, 2097152.0, 1229.0]
    L3 = plan.Layer(4, 16, 1024, 1024, 2, 1.2, False, "gated3", 8, 2)
    v3 = plan.derive_volumes(L3, (32, 8, 2, 4, 8, 4))
    assert v3[4] == 3 and v3[3] == v[3] and abs(v3[5] - (1572864.0 + 1048576.0)) < 1e-6
    with pytest.raises(ConfigError, match="experts must divide evenly"):
        plan.derive_volumes(L, (32, 8, 2, 4, 3, 4))
    with pytest.raises(ConfigError, match="layer: batch must be positive"):
        plan.capacity_tokens(plan.Layer(0, 1, 1, 1, 1))


def test_optimizer_kats():
    # test_pipeline_optimizer.cpp:160-228, 308-329
    d = plan.find_degree(REF_VOL, REF_PROFILE, 0.0, 1, 16)
    assert int(d[0]) == 4 and int(d[1]) == 3 and abs(d[2] - 25.2) < 1e-12 and d[10] == 0
    p = plan.plan_layer(REF_VOL, REF_PROFILE, 3.0, 4)
    assert (p["r_fwd"], p["case_fwd"], p["r_bwd"], p["case_bwd"]) == (4, 3, 4, 2)
    assert abs(p["t_moe_fwd_ms"] - 25.2) < 1e-12 and abs(p["t_moe_bwd_ms"] - 43.2) < 1e-12
    assert abs(p["t_olp_moe_bwd_ms"] - 19.2) < 1e-12


def test_schedule_baseline_kats():
    # test_schedule_sim.cpp:33-51, 197-210
    pr = prof((1.0, 1e-6), (0.1, 1e-7), (0.1, 1e-7), (0.5, 1e-6), (0.01, 1e-9))
    vol = np.array([1e6, 1e6, 1e6, 1e6, 2, 0, 0], dtype=float)
    want = {"fsmoe": 6.3, "fsmoe_no_iio": 6.621, "pipemoe": 6.6, "sequential": 6.642}
    for style, ms in want.items():
        out = plan.simulate_stage(vol, pr, 1, 2, style=style)
        assert abs(out[0] - ms) < 1e-12, (style, out[0])
    r1 = plan.simulate_stage(vol, pr, 1, 1)
    assert abs(r1[0] - (2.0 + 0.2 + 0.022 + 0.2 + 2.0)) < 1e-12


def test_partition_kats():
    # test_grad_partition.cpp:69-77, 195-210
    pr = prof((1.0, 1e-6), (0.1, 1e-6), (0.1, 1e-6), (0.0, 1e-6), (0.25, 1e-9))
    out = plan.build_partition_plan([(REF_VOL, 2.0, 1.5e7), (REF_VOL, 2.0, 0.0)], pr,
                                    de=(0, 200, 0.8, 0.9, 1), r_max=4)
    # layer 0 / layer 1 rows of 9, then tail, tail_ms, objective, step2_ran
    assert out[9 * 2 + 3] == 0.0 and out[9 * 2] == 0.0  # no optimizer, no tail
    assert abs(out[9 + 1] - 2e6) < 1e-6 and abs(out[9 + 2] - 1.3e7) < 1e-3
    assert abs(out[9 + 4] - 15.0) < 1e-12 and abs(out[9 + 7] - 19.2) < 1e-12
    assert int(out[5]) == 4 and int(out[6]) == 2  # sync_window degree/case of layer 0


def test_pipeline_chunks_cover_capacity():
    for C in (1, 100, 128, 1000, 1024, 8192, 1229):
        for r in (1, 2, 3, 4, 7, 16):
            ch = plan.pipeline_chunks(C, r)
            assert ch[0][0] == 0 and ch[-1][1] == C
            assert all(a < b for a, b in ch)
            assert all(ch[i][1] == ch[i + 1][0] for i in range(len(ch) - 1))
            assert all(a % 128 == 0 for a, _ in ch)
            assert len(ch) == min(r, (C + 127) // 128)


# ------------------------------------------------- randomized ref parity --

def _rand_profile(rng, symmetric):
    u = lambda lo, hi: rng.uniform(lo, hi)  # noqa: E731
    a2a = (u(0.02, 0.6), u(5e-8, 5e-6))
    ag = (u(0.02, 0.6), u(5e-8, 5e-6))
    rs = ag if symmetric else (u(0.02, 0.6), u(5e-8, 5e-6))
    return prof(a2a, ag, rs, (u(0.05, 0.8), u(1e-7, 6e-6)), (u(0.02, 0.15), u(5e-12, 1e-10)))


def _rand_layer(rng):
    L = plan.Layer(batch=int(rng.choice([1, 2, 4])), heads=16, seq_len=int(rng.choice([512, 1024, 2048])),
                   model_dim=int(rng.choice([1024, 2048, 4096])), hidden_scale=int(rng.choice([2, 3, 4])),
                   capacity_factor=float(rng.choice([1.2, 2.4])), experts=int(rng.choice([6, 8])),
                   top_k=int(rng.choice([1, 2])), ffn=str(rng.choice(["simple", "gated3"])))
    par = tuple(int(v) for v in rng.choice([(8, 8, 1, 1, 2, 1), (16, 8, 2, 1, 2, 4), (32, 8, 1, 2, 2, 2)]))
    return L, par


@needs_ref
def test_volumes_match_reference():
    rng = np.random.default_rng(1)
    R = ref()
    for _ in range(60):
        L, par = _rand_layer(rng)
        ints, dbls = L.arrays()
        assert plan.capacity_tokens(L) == R.capacity_tokens(ints, dbls)
        assert np.array_equal(plan.derive_volumes(L, par), R.derive_volumes(ints, dbls, par))


@needs_ref
@pytest.mark.parametrize("symmetric", [True, False])
def test_optimizer_matches_reference(symmetric):
    rng = np.random.default_rng(2 + symmetric)
    R = ref()
    for _ in range(80):
        L, par = _rand_layer(rng)
        vol = plan.derive_volumes(L, par)
        pr = _rand_profile(rng, symmetric)
        t_gar = float(rng.choice([0.0, rng.uniform(0.05, 5.0)]))
        for mult in (1, 2):
            assert np.array_equal(plan.find_degree(vol, pr, t_gar, mult, 16),
                                  R.find_degree(vol, pr, t_gar, mult, 16))
        p = plan.plan_layer(vol, pr, t_gar, 16)
        r = R.plan_layer(vol, pr, t_gar, 16)
        assert [p["r_fwd"], p["case_fwd"], p["t_moe_fwd_ms"], p["boundary_fwd"], p["r_bwd"],
                p["case_bwd"], p["t_moe_bwd_ms"], p["boundary_bwd"], p["t_gar_bwd_ms"],
                p["t_olp_moe_bwd_ms"]] == list(r)


@needs_ref
def test_simulator_matches_reference():
    rng = np.random.default_rng(5)
    R = ref()
    for _ in range(40):
        L, par = _rand_layer(rng)
        vol = plan.derive_volumes(L, par)
        pr = _rand_profile(rng, bool(rng.integers(2)))
        r = int(rng.integers(1, 9))
        sync = [float(v) for v in rng.uniform(0.1, 3.0, int(rng.integers(0, 3)))]
        for style, sid in plan.STYLES.items():
            mult = int(rng.integers(1, 3))
            assert np.array_equal(plan.simulate_stage(vol, pr, mult, r, sync, style),
                                  R.simulate_stage(vol, pr, mult, r, sync, sid))
        assert plan.brute_force_degree(vol, pr, 1.0, 2, 12) == R.brute_force_degree(vol, pr, 1.0, 2, 12)


@needs_ref
def test_fit_matches_reference():
    rng = np.random.default_rng(7)
    R = ref()
    for _ in range(30):
        samples = []
        for kind in ("a2a", "ag", "rs", "ar", "gemm"):
            a, b = rng.uniform(-0.1, 0.5), rng.uniform(-1e-7, 1e-6)
            for n in rng.uniform(1e5, 1e7, int(rng.integers(2, 8))):
                samples.append((kind, float(n), float(a + b * n + rng.normal(0, 0.01))))
        p, m, c = plan.fit_profile(samples, 0.0)
        rp, rm, rc = R.fit_profile([plan.KINDS[k] for k, _, _ in samples],
                                   [s[1] for s in samples], [s[2] for s in samples], 0.0)
        assert np.array_equal(p, rp) and m == rm and c == rc


@needs_ref
def test_partition_matches_reference():
    rng = np.random.default_rng(11)
    R = ref()
    for trial in range(6):
        pr = _rand_profile(rng, True)
        layers = []
        for _ in range(int(rng.integers(1, 4))):
            L, par = _rand_layer(rng)
            vol = plan.derive_volumes(L, par)
            layers.append((vol, float(rng.uniform(0, 3)), float(rng.uniform(0, 3e7))))
        de = (0, 25, 0.8, 0.9, 100 + trial)
        flat = np.concatenate([np.concatenate([np.asarray(v, float), [d, g]]) for v, d, g in layers])
        assert np.array_equal(plan.build_partition_plan(layers, pr, de, 8),
                              R.build_partition_plan(flat, len(layers), pr, de, 8))


@needs_ref
def test_error_messages_match_reference():
    R = ref()
    # unknown kind / missing kind / fit quality
    with pytest.raises(ConfigError) as e:
        plan.fit_profile([("a2a", 1.0, 1.0), ("a2a", 2.0, 2.0)])
    with pytest.raises(pyoracle.OracleError) as r:
        R.fit_profile([0, 0], [1.0, 2.0], [1.0, 2.0], 0.0)
    assert str(e.value) == str(r.value)
