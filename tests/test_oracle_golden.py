"""Pins the CPU oracle (oracle/fsmoe_oracle.c, the plain-C restatement of
proj/src/workload.cpp) before anything is compared against it:

* bit-identical to the golden vectors the REFERENCE produced
  (tests/golden/, oracle/gen_golden.py over oracle/_ref);
* bit-identical to the reference itself on fresh random instances when the
  reference build is present;
* the reference test suites' known-answer tests, restated
  (proj/tests/test_workload.cpp, proj/tests/acceptance.cpp:459-610);
* the config-1 fingerprint (dropped / fill match the
  survey, hashes re-derived from the reference).
CPU only.
"""
import json
import os

import numpy as np
import pytest

import fingerprint
import gen_golden
import pyoracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = json.load(open(os.path.join(GOLD, "routing_cases.json")))["cases"]
NPZ = np.load(os.path.join(GOLD, "routing_cases.npz"))


def arr(i, k):
    n = f"c{i}_{k}"
    return NPZ[n] if n in NPZ.files else None


@pytest.fixture(scope="module")
def port():
    return pyoracle.Oracle("port")


@pytest.mark.parametrize("i", range(len(CASES)))
def test_port_matches_reference_golden(port, i):
    c = CASES[i]
    if c["inputs_stored"]:
        x, ws, wn, pj = arr(i, "x"), arr(i, "w_score"), arr(i, "w_noise"), arr(i, "proj")
    else:
        x, ws, wn, pj = gen_golden.case_inputs(c["seed"], c["gate"], c["T"], c["M"], c["E"], c["k"],
                                               c["proj_dim"], c["suppress_noise"], c["ties"])
    g = port.run_gate(c["gate"], c["k"], c["gate_seed"], x, ws, wn, pj)
    np.testing.assert_array_equal(g.token, arr(i, "pick_token"))
    np.testing.assert_array_equal(g.expert, arr(i, "pick_expert"))
    np.testing.assert_array_equal(g.weight, arr(i, "pick_weight"))  # same host libm: bit-exact
    d = port.dispatch(x, c["E"], g.token, g.expert, c["capacity"])
    np.testing.assert_array_equal(d.slot_of_pick, arr(i, "slot_of_pick"))
    np.testing.assert_array_equal(d.fill, arr(i, "fill"))
    assert d.dropped == int(arr(i, "dropped")[0])
    if c["inputs_stored"]:
        y = port.combine(d.buffers, c["T"], c["E"], g.token, g.expert, g.weight, d.slot_of_pick, c["M"])
        np.testing.assert_array_equal(y, arr(i, "y"))


def test_port_error_messages_match_reference_golden(port):
    errs = json.load(open(os.path.join(GOLD, "errors.json")))
    for e in errs:
        got = gen_golden.run_error(port, e["kind"], e["args"])
        assert got["code"] == e["code"] and got["message"] == e["message"], e["name"]


def test_fingerprint_config1(port):
    for gate, want in fingerprint.EXPECTED.items():
        assert fingerprint.run(gate, port) == want, gate
    golden = json.load(open(os.path.join(GOLD, "fingerprint.json")))["values"]
    for gate, want in golden.items():
        assert list(fingerprint.EXPECTED[gate]) == want


@pytest.mark.skipif(not pyoracle.available("reference"), reason="reference not built")
def test_port_matches_reference_on_random_instances(port):
    ref = pyoracle.Oracle("reference")
    rng = np.random.default_rng(123)
    for trial in range(40):
        gate = ["noisy_topk", "sigmoid_topk", "cosine_topk", "expert_choice"][trial % 4]
        T, M, E = int(rng.integers(2, 300)), int(rng.integers(2, 64)), int(rng.integers(2, 24))
        k = int(rng.integers(1, T + 1)) if gate == "expert_choice" else int(rng.integers(1, E + 1))
        P = int(rng.integers(1, 12))
        x = rng.uniform(-1, 1, (T, M))
        ws = rng.uniform(-1, 1, (P if gate == "cosine_topk" else M, E))
        wn = rng.uniform(-1, 1, (M, E))
        pj = rng.uniform(-1, 1, (P, M))
        a = port.run_gate(gate, k, trial, x, ws, wn, pj)
        b = ref.run_gate(gate, k, trial, x, ws, wn, pj)
        for f in ("token", "expert", "weight"):
            np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
        cap = int(rng.integers(1, max(2, T)))
        da = port.dispatch(x, E, a.token, a.expert, cap)
        db = ref.dispatch(x, E, b.token, b.expert, cap)
        np.testing.assert_array_equal(da.buffers, db.buffers)
        np.testing.assert_array_equal(da.slot_of_pick, db.slot_of_pick)
        ya = port.combine(da.buffers, T, E, a.token, a.expert, a.weight, da.slot_of_pick, M)
        yb = ref.combine(db.buffers, T, E, b.token, b.expert, b.weight, db.slot_of_pick, M)
        np.testing.assert_array_equal(ya, yb)


# ------------------------------------------- reference test-suite KATs ----

def _brute_topk(scores, k):
    idx = sorted(range(len(scores)), key=lambda i: (-scores[i], i))[:k]
    return sorted(idx)


def _softmax(scores, keep):
    mx = max(scores[i] for i in keep)
    z = sum(np.exp(scores[i] - mx) for i in keep)
    return [np.exp(scores[i] - mx) / z for i in keep]


def test_kat_noise_suppressed_noisy_gate(port):
    """test_workload.cpp:160-191 (seed 11): with x > 0 and W_noise = -1e4 the
    noise scale is exactly 0, so the gate equals plain softmax-top-k."""
    rng = pyoracle.MtRng(11)
    for _ in range(300):
        T, E, M = 2 + rng.next() % 5, 2 + rng.next() % 5, 2 + rng.next() % 4
        k = 1 + rng.next() % min(3, E)
        x = rng.matrix(T, M, 0.2, 1.5)
        ws = rng.matrix(M, E, -1.0, 1.0)
        wn = np.full((M, E), -1e4)
        g = port.run_gate("noisy_topk", k, 99, x, ws, wn)
        assert g.token.size == T * k
        for t in range(T):
            logits = x[t] @ ws
            keep = _brute_topk(logits, k)
            assert list(g.expert[t * k:(t + 1) * k]) == keep
            np.testing.assert_allclose(g.weight[t * k:(t + 1) * k], _softmax(logits, keep), rtol=1e-12)


def test_kat_small_gates(port):
    # ties -> lowest index (test_workload.cpp:215-227)
    g = port.run_gate("sigmoid_topk", 2, 0, np.array([[1.0]]), np.array([[1.0, 1.0, 0.0]]))
    assert list(g.expert) == [0, 1]
    # sigmoid weights (229-262)
    g = port.run_gate("sigmoid_topk", 1, 0, np.array([[1.0]]), np.array([[0.0, -5.0]]))
    assert g.expert[0] == 0 and g.weight[0] == 0.5
    g = port.run_gate("sigmoid_topk", 2, 0, np.array([[1.0]]), np.array([[-1.0, 4.0]]))
    np.testing.assert_allclose(g.weight, [1 / (1 + np.exp(1.0)), 1 / (1 + np.exp(-4.0))])
    # cosine (289-323)
    pj = np.eye(2)
    g = port.run_gate("cosine_topk", 1, 0, np.array([[3.0, 0.0]]), np.array([[0.5, 0.0], [0.0, 2.0]]), None, pj)
    assert g.expert[0] == 0 and g.weight[0] == 1.0
    with pytest.raises(pyoracle.OracleError, match="expert embedding has zero norm"):
        port.run_gate("cosine_topk", 1, 0, np.array([[1.0, 0.0]]), np.zeros((2, 1)), None, pj)
    # expert choice (366-394)
    x = np.eye(2)
    ws = np.array([[9.0, 0.0], [0.0, 9.0]])
    g = port.run_gate("expert_choice", 1, 0, x, ws)
    assert list(g.token) == [0, 1] and list(g.expert) == [0, 1] and g.weight[0] == 1.0
    assert port.run_gate("expert_choice", 2, 0, x, ws).token.size == 4
    with pytest.raises(pyoracle.OracleError, match="expert capacity exceeds token count"):
        port.run_gate("expert_choice", 3, 0, x, ws)


def test_kat_dispatch_combine(port):
    # test_workload.cpp:427-512
    x = np.array([[3.0], [7.0]])
    d = port.dispatch(x, 2, [0, 1], [0, 1], 1)
    assert d.dropped == 0 and list(d.buffers[:, 0]) == [3.0, 7.0] and list(d.fill) == [1, 1]
    d = port.dispatch(x, 2, [0, 1], [0, 0], 1)
    assert d.dropped == 1 and list(d.buffers[:, 0]) == [3.0, 0.0] and list(d.slot_of_pick) == [0, -1]
    x3 = np.array([[t * 10.0 + j for j in range(2)] for t in range(3)])
    d = port.dispatch(x3, 3, [0, 1, 2], [2, 0, 1], 1)
    y = port.combine(d.buffers, 3, 3, [0, 1, 2], [2, 0, 1], [1.0, 1.0, 1.0], d.slot_of_pick, 2)
    np.testing.assert_array_equal(y, x3)
    x = np.array([[5.0], [6.0]])
    d = port.dispatch(x, 1, [0, 1], [0, 0], 1)
    y = port.combine(d.buffers, 2, 1, [0, 1], [0, 0], [1.0, 1.0], d.slot_of_pick, 1)
    assert list(y[:, 0]) == [5.0, 0.0]


def test_kat_identity_combine(port):
    """test_workload.cpp:456-483 (seed 41): identity experts scale each token by
    the sum of its surviving weights."""
    rng = pyoracle.MtRng(41)
    for _ in range(100):
        T, E, M = 2 + rng.next() % 5, 2 + rng.next() % 4, 2 + rng.next() % 4
        k = 1 + rng.next() % 2
        x = rng.matrix(T, M, -1, 1)
        ws = rng.matrix(M, E, -1, 1)
        g = port.run_gate("sigmoid_topk", k, 0, x, ws)
        cap = 1 + rng.next() % T
        d = port.dispatch(x, E, g.token, g.expert, cap)
        assert (d.fill <= cap).all()
        y = port.combine(d.buffers, T, E, g.token, g.expert, g.weight, d.slot_of_pick, M)
        wsum = np.zeros(T)
        for p in range(g.token.size):
            if d.slot_of_pick[p] >= 0:
                wsum[g.token[p]] += g.weight[p]
        np.testing.assert_allclose(y, wsum[:, None] * x, rtol=1e-12, atol=1e-15)
