"""TEST INFRASTRUCTURE ONLY — generates tests/golden/ from the REFERENCE.

Runs the reference's own run_gate -> dispatch_tokens -> combine_tokens,
compiled from /root/reference/proj/src by oracle/Makefile into
oracle/_ref/libfsmoe_ref.so, on seeded inputs and stores inputs and outputs
as small fixtures. /root/reference does not exist on the GPU box, so the
fixtures (not the reference) are what travel.

Fixtures written:
  tests/golden/routing_cases.npz   per-case inputs + reference outputs
  tests/golden/routing_cases.json  case metadata (shapes, gate, seed, capacity)
  tests/golden/errors.json         ConfigError messages for invalid inputs
  tests/golden/fingerprint.json    Appendix-C config-1 fingerprint

Usage: python oracle/gen_golden.py   (needs make -C oracle ref)
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import fingerprint  # noqa: E402
import pyoracle  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden")


def case_inputs(seed, gate, T, M, E, k, proj_dim=0, suppress_noise=False, ties=False):
    """Inputs drawn from one mt19937_64(seed) stream (x, w_score, w_noise, proj)."""
    rng = pyoracle.MtRng(seed)
    lo = 0.2 if suppress_noise else -1.0
    hi = 1.5 if suppress_noise else 1.0
    if gate == "cosine_topk":
        lo, hi = 0.1, 1.0
    x = rng.matrix(T, M, lo, hi)
    rows = proj_dim if gate == "cosine_topk" else M
    ws = rng.matrix(rows, E, -1.0, 1.0) if gate != "cosine_topk" else rng.matrix(rows, E, 0.1, 1.0)
    wn = rng.matrix(M, E, -0.5, 0.5)
    if suppress_noise:
        wn[:] = -1e4
    pj = rng.matrix(proj_dim, M, 0.1, 1.0) if proj_dim else np.zeros((0, 0))
    if ties:
        # duplicate expert columns -> exact score ties that must break low
        for e in range(1, E, 2):
            ws[:, e] = ws[:, e - 1]
        if gate == "noisy_topk":
            for e in range(1, E, 2):
                wn[:, e] = wn[:, e - 1]
    return x, ws, wn, pj


CASES = []


def add(gate, T, M, E, k, cap, seed, proj_dim=0, suppress=False, ties=False, gseed=None):
    CASES.append(dict(gate=gate, T=T, M=M, E=E, k=k, capacity=cap, seed=seed,
                      proj_dim=proj_dim, suppress_noise=suppress, ties=ties,
                      gate_seed=seed * 7 + 3 if gseed is None else gseed))


def build_case_list():
    s = 100
    for gate in ("noisy_topk", "sigmoid_topk", "cosine_topk"):
        for (T, M, E, k) in [(8, 4, 4, 2), (33, 16, 5, 1), (64, 32, 8, 2), (100, 24, 6, 3),
                             (257, 64, 16, 1), (512, 128, 8, 2), (300, 40, 64, 4)]:
            for capmode in ("tight", "exact", "loose"):
                s += 1
                exact = -(-k * T // E)
                cap = {"tight": max(1, exact // 2), "exact": exact, "loose": T * k}[capmode]
                add(gate, T, M, E, k, cap, s, proj_dim=(8 if gate == "cosine_topk" else 0))
        # ties
        s += 1
        add(gate, 40, 12, 6, 2, 10, s, proj_dim=(4 if gate == "cosine_topk" else 0), ties=True)
    # noise suppressed (test_workload.cpp:160-191 style)
    for T, M, E, k in [(16, 4, 5, 2), (128, 32, 8, 2), (77, 9, 7, 3)]:
        s += 1
        add("noisy_topk", T, M, E, k, -(-k * T // E), s, suppress=True)
    # expert choice: caps 1, T/2, T ; dispatch capacities tight/exact
    for (T, M, E) in [(8, 4, 4), (64, 32, 8), (300, 40, 6), (1024, 64, 16)]:
        for c in sorted({1, max(1, T // 4), T // 2, T}):
            for dcap in sorted({c, max(1, c // 2)}):
                s += 1
                add("expert_choice", T, M, E, c, dcap, s)
    s += 1
    add("expert_choice", 40, 12, 6, 10, 10, s, ties=True)
    # k == E, k == 1
    s += 1
    add("sigmoid_topk", 50, 10, 4, 4, 50, s)
    s += 1
    add("noisy_topk", 50, 10, 4, 4, 30, s)


def run_case(orc, c):
    x, ws, wn, pj = case_inputs(c["seed"], c["gate"], c["T"], c["M"], c["E"], c["k"],
                                c["proj_dim"], c["suppress_noise"], c["ties"])
    g = orc.run_gate(c["gate"], c["k"], c["gate_seed"], x, ws, wn, pj)
    d = orc.dispatch(x, c["E"], g.token, g.expert, c["capacity"])
    y = orc.combine(d.buffers, c["T"], c["E"], g.token, g.expert, g.weight,
                    d.slot_of_pick, c["M"])
    return dict(x=x, w_score=ws, w_noise=wn, proj=pj, pick_token=g.token,
                pick_expert=g.expert, pick_weight=g.weight, slot_of_pick=d.slot_of_pick,
                fill=d.fill, dropped=np.array([d.dropped]), buffers=d.buffers, y=y)


ERROR_CASES = [
    # (name, call, args) -> reference message
    ("gate_empty", "gate", dict(gate="sigmoid_topk", T=0, M=3, E=2, k=1)),
    ("gate_no_experts", "gate", dict(gate="sigmoid_topk", T=2, M=3, E=0, k=1)),
    ("gate_k_zero", "gate", dict(gate="sigmoid_topk", T=2, M=3, E=2, k=0)),
    ("gate_k_gt_E", "gate", dict(gate="noisy_topk", T=2, M=3, E=2, k=3)),
    ("gate_ec_cap_gt_T", "gate", dict(gate="expert_choice", T=2, M=3, E=2, k=3)),
    ("gate_noisy_noise_dims", "gate", dict(gate="noisy_topk", T=2, M=3, E=2, k=1, wn_rows=2)),
    ("gate_sigmoid_dims", "gate", dict(gate="sigmoid_topk", T=2, M=3, E=2, k=1, ws_rows=4)),
    ("gate_ec_dims", "gate", dict(gate="expert_choice", T=2, M=3, E=2, k=1, ws_rows=4)),
    ("gate_cos_proj_dims", "gate", dict(gate="cosine_topk", T=2, M=3, E=2, k=1, P=2, pj_cols=4)),
    ("gate_cos_score_dims", "gate", dict(gate="cosine_topk", T=2, M=3, E=2, k=1, P=2, ws_rows=3)),
    ("gate_cos_zero_token", "gate", dict(gate="cosine_topk", T=3, M=3, E=2, k=1, P=2, zero_token=1)),
    ("gate_cos_zero_token0", "gate", dict(gate="cosine_topk", T=3, M=3, E=2, k=1, P=2, zero_token=0,
                                          zero_expert=1)),
    ("gate_cos_zero_expert", "gate", dict(gate="cosine_topk", T=3, M=3, E=2, k=1, P=2, zero_expert=1)),
    ("dispatch_cap_zero", "dispatch", dict(cap=0)),
    ("dispatch_bad_expert", "dispatch", dict(cap=2, bad="expert")),
    ("dispatch_bad_token", "dispatch", dict(cap=2, bad="token")),
    ("combine_width", "combine", dict(width=3, model_dim=4)),
    ("combine_layout", "combine", dict(width=4, model_dim=4, short=True)),
]


def error_inputs(kind, a):
    """Deterministic small inputs for the error cases (also used by the tests)."""
    if kind == "gate":
        T, M, E, k = a["T"], a["M"], a["E"], a["k"]
        P = a.get("P", 0)
        x = np.arange(1, T * M + 1, dtype=np.float64).reshape(T, M) / 7.0 if T * M else np.zeros((T, M))
        ws_rows = a.get("ws_rows", P if a["gate"] == "cosine_topk" else M)
        ws = np.ones((ws_rows, E)) * 0.5 if E else np.zeros((ws_rows, 0))
        wn = np.ones((a.get("wn_rows", M), E)) * 0.1 if E else np.zeros((M, 0))
        pj = np.ones((P, a.get("pj_cols", M))) * 0.3 if P else np.zeros((0, 0))
        if "zero_token" in a:
            x[a["zero_token"], :] = 0.0
        if "zero_expert" in a:
            ws[:, a["zero_expert"]] = 0.0
        return dict(gate=a["gate"], k=k, x=x, w_score=ws, w_noise=wn, proj=pj)
    if kind == "dispatch":
        x = np.arange(8, dtype=np.float64).reshape(4, 2)
        tok = np.array([0, 1, 2, 3], np.int32)
        exp = np.array([0, 1, 0, 1], np.int32)
        if a.get("bad") == "expert":
            exp[2] = 5
        if a.get("bad") == "token":
            tok[3] = 9
        return dict(x=x, E=2, pick_token=tok, pick_expert=exp, capacity=a["cap"])
    if kind == "combine":
        buf = np.ones((4, a["width"]))
        tok = np.array([0, 1], np.int32)
        exp = np.array([0, 1], np.int32)
        w = np.array([0.5, 0.25])
        slots = np.array([0, 2], np.int32) if not a.get("short") else np.array([0], np.int32)
        return dict(buffers=buf, T=2, E=2, pick_token=tok, pick_expert=exp, pick_weight=w,
                    slot_of_pick=slots, model_dim=a["model_dim"])
    raise ValueError(kind)


def run_error(orc, kind, a):
    inp = error_inputs(kind, a)
    try:
        if kind == "gate":
            orc.run_gate(inp["gate"], inp["k"], 1, inp["x"], inp["w_score"], inp["w_noise"], inp["proj"])
        elif kind == "dispatch":
            orc.dispatch(inp["x"], inp["E"], inp["pick_token"], inp["pick_expert"], inp["capacity"])
        else:
            orc.combine(inp["buffers"], inp["T"], inp["E"], inp["pick_token"], inp["pick_expert"],
                        inp["pick_weight"], inp["slot_of_pick"], inp["model_dim"])
    except pyoracle.OracleError as e:
        return dict(code=e.code, message=str(e))
    return dict(code=0, message="")


def main():
    if not pyoracle.available("reference"):
        sys.exit("reference oracle not built: make -C oracle ref")
    orc = pyoracle.Oracle("reference")
    os.makedirs(OUT, exist_ok=True)
    build_case_list()
    arrays = {}
    for i, c in enumerate(CASES):
        r = run_case(orc, c)
        c["n_picks"] = int(r["pick_token"].size)
        c["dropped"] = int(r["dropped"][0])
        small = c["T"] * c["M"] <= 8192
        c["inputs_stored"] = small
        for key, v in r.items():
            # buffers are a pure gather of x (checked via slot_of_pick); large
            # inputs/outputs are regenerated from the seed with the C port.
            if key == "buffers" or (not small and key in ("x", "y", "w_noise", "w_score", "proj")):
                continue
            arrays[f"c{i}_{key}"] = v
    np.savez_compressed(os.path.join(OUT, "routing_cases.npz"), **arrays)
    with open(os.path.join(OUT, "routing_cases.json"), "w") as f:
        json.dump(dict(generator="oracle/gen_golden.py", backend="reference (oracle/_ref)",
                       cases=CASES), f, indent=1)
    errs = []
    for name, kind, a in ERROR_CASES:
        errs.append(dict(name=name, kind=kind, args=a, **run_error(orc, kind, a)))
    with open(os.path.join(OUT, "errors.json"), "w") as f:
        json.dump(errs, f, indent=1)
    fp = {gate: list(fingerprint.run(gate, orc)) for gate in fingerprint.EXPECTED}
    with open(os.path.join(OUT, "fingerprint.json"), "w") as f:
        json.dump(dict(recipe=fingerprint.__doc__, backend="reference (oracle/_ref)", values=fp), f,
                  indent=1)
    print(f"{len(CASES)} cases, {len(errs)} error cases -> {OUT}")


if __name__ == "__main__":
    main()
