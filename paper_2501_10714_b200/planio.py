"""Planner interchange formats and the planner command line (SURVEY.md §8f
row 4): the reference's profile / model / plan JSON documents and bench CSV
(json_io.cpp:49-245, 278-328) and its `fit | plan | simulate | compare`
subcommands (cli/main.cpp:79-291), over this package's bit-exact planner
port (plan.py -> libfsmoe.so). A profile fitted on the box by autotune.py can
be saved here and read by the reference's tools, and the other way round.

Documents keep the reference's key order (its `json` is nlohmann::ordered_json,
json_io.hpp:16) with dump(2)'s two-space indent; tests/test_planio.py checks
them byte for byte against documents the reference itself wrote. Validation
errors raise ConfigError with the reference's messages; the CLI maps
ConfigError / FitQualityError / InvariantError to exit codes 2 / 3 / 4
(common.hpp:9-14, main.cpp:363-375).

    python -m paper_2501_10714_b200.planio fit --bench b.csv [--out p.json] [--min-r2 0.99]
    python -m paper_2501_10714_b200.planio plan --model m.json --profile p.json [--r-max R] [--seed S]
    python -m paper_2501_10714_b200.planio simulate --model m.json --profile p.json [--pass bwd] ...
    python -m paper_2501_10714_b200.planio compare a.json b.json [--tol 1e-9]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import re
import sys

import numpy as np

from . import _native as NL
from . import plan as P

KIND_ORDER = ("a2a", "ag", "rs", "ar", "gemm")   # ClusterProfile members, cost_models.hpp:46-53
RESOURCES = ("inter", "intra", "compute")        # schedule_sim.cpp:41-48


def _err(msg):
    return NL.ConfigError(2, msg)


# --- field readers with the reference's messages (json_io.cpp:12-33) -------

def _require(j, key, where):
    if not isinstance(j, dict) or key not in j:
        raise _err(f"{where}: missing field '{key}'")
    return j[key]


def _number(j, key, where):
    v = _require(j, key, where)
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        raise _err(f"{where}: field '{key}' must be a number")
    return float(v)


def _integer(j, key, where):
    v = _require(j, key, where)
    if isinstance(v, bool) or not isinstance(v, int):
        raise _err(f"{where}: field '{key}' must be an integer")
    return int(v)


def dumps(doc) -> str:
    """dump(2) layout: insertion order, two-space indent, trailing newline."""
    return json.dumps(doc, indent=2) + "\n"


def _parse_json(text, path):
    try:
        return json.loads(text)
    except json.JSONDecodeError as e:
        raise _err(f"{path}: {e}") from None


def read_text_file(path) -> str:
    try:
        with open(path, "rb") as f:
            return f.read().decode()
    except OSError:
        raise _err(f"cannot read {path}") from None


def write_text_file(path, text: str) -> None:
    try:
        with open(path, "wb") as f:
            f.write(text.encode())
    except OSError:
        raise _err(f"cannot write {path}") from None


# --- profile (json_io.cpp:49-80) -------------------------------------------

def profile_to_json(profile) -> dict:
    """profile: the planner's 10-double array (alpha, beta per kind)."""
    p = np.asarray(profile, dtype=np.float64)
    return {k: {"alpha_ms": float(p[2 * i]), "beta_ms_per_unit": float(p[2 * i + 1])}
            for i, k in enumerate(KIND_ORDER)}


def profile_from_json(j) -> np.ndarray:
    out = np.zeros(10)
    for i, k in enumerate(KIND_ORDER):
        m = _require(j, k, "profile")
        out[2 * i] = _number(m, "alpha_ms", f"profile.{k}")
        out[2 * i + 1] = _number(m, "beta_ms_per_unit", f"profile.{k}")
    return out


def load_profile(path) -> np.ndarray:
    return profile_from_json(_parse_json(read_text_file(path), path))


def save_profile(profile, path) -> None:
    write_text_file(path, dumps(profile_to_json(profile)))


# --- layer / parallel / model (json_io.cpp:82-196) -------------------------

def layer_to_json(l: P.Layer) -> dict:
    j = {"batch": l.batch, "heads": l.heads, "seq_len": l.seq_len, "model_dim": l.model_dim,
         "hidden_scale": l.hidden_scale,
         "capacity_factor": "*" if l.unlimited else float(l.capacity_factor),
         "ffn": "gated3" if l.ffn == "gated3" else "simple", "experts": l.experts,
         "top_k": l.top_k, "t_olp_dense_ms": float(l.t_olp_dense_ms)}
    if l.grad_override is not None:
        j["grad_elements"] = float(l.grad_override)
    return j


def layer_from_json(j) -> P.Layer:
    w = "layer"
    kw = {k: _integer(j, k, w) for k in ("batch", "heads", "seq_len", "model_dim", "hidden_scale")}
    f = _require(j, "capacity_factor", w)
    if isinstance(f, str):
        if f != "*":
            raise _err('layer: capacity_factor must be a number or "*"')
        kw["unlimited"] = True
    elif isinstance(f, (int, float)) and not isinstance(f, bool):
        kw["capacity_factor"] = float(f)
    else:
        raise _err('layer: capacity_factor must be a number or "*"')
    ffn = _require(j, "ffn", w)
    if ffn not in ("simple", "gated3"):
        raise _err(f"layer: unknown ffn '{ffn}'")
    kw["ffn"] = ffn
    kw["experts"] = _integer(j, "experts", w)
    kw["top_k"] = _integer(j, "top_k", w)
    if "t_olp_dense_ms" in j:
        kw["t_olp_dense_ms"] = _number(j, "t_olp_dense_ms", w)
    if "grad_elements" in j:
        kw["grad_override"] = _number(j, "grad_elements", w)
    return P.Layer(**kw)


PARALLEL_KEYS = ("total_gpus", "gpus_per_node", "data_parallel", "tensor_parallel",
                 "expert_parallel", "expert_shard")


def parallel_to_json(par) -> dict:
    """par: (total_gpus, gpus_per_node, dp, tp, ep, esp) as plan.derive_volumes takes."""
    return dict(zip(PARALLEL_KEYS, map(int, par)))


def parallel_from_json(j) -> tuple:
    return tuple(_integer(j, k, "parallel") for k in PARALLEL_KEYS)


DE_DEFAULT = (0, 200, 0.8, 0.9, 1)  # DeParams, grad_partition.hpp:20-26


def model_from_json(j) -> dict:
    """-> {"parallel": tuple, "layers": [Layer], "r_max": int, "de": tuple}."""
    m = {"parallel": parallel_from_json(_require(j, "parallel", "model"))}
    layers = _require(j, "layers", "model")
    if not isinstance(layers, list) or not layers:
        raise _err("model: 'layers' must be a non-empty array")
    m["layers"] = [layer_from_json(l) for l in layers]
    m["r_max"] = _integer(j, "r_max", "model") if "r_max" in j else 16
    de = list(DE_DEFAULT)
    if "de" in j:
        d = j["de"]
        for i, (k, rd) in enumerate((("population", _integer), ("generations", _integer),
                                     ("weight", _number), ("crossover", _number))):
            if k in d:
                de[i] = rd(d, k, "model.de")
        if "seed" in d:
            s = _require(d, "seed", "model.de")
            if isinstance(s, bool) or not isinstance(s, int) or s < 0:
                raise _err("model.de: field 'seed' must be an unsigned integer")
            de[4] = s
    m["de"] = tuple(de)
    return m


def model_to_json(m) -> dict:
    pop, gens, w, cr, seed = m["de"]
    return {"parallel": parallel_to_json(m["parallel"]),
            "layers": [layer_to_json(l) for l in m["layers"]], "r_max": int(m["r_max"]),
            "de": {"population": int(pop), "generations": int(gens), "weight": float(w),
                   "crossover": float(cr), "seed": int(seed)}}


def load_model(path) -> dict:
    return model_from_json(_parse_json(read_text_file(path), path))


# --- plans (json_io.cpp:198-245; main.cpp:58-68) ---------------------------

def plan_to_json(p: dict) -> dict:
    keys = ("r_fwd", "case_fwd", "t_moe_fwd_ms", "boundary_fwd", "r_bwd", "case_bwd",
            "t_moe_bwd_ms", "boundary_bwd", "t_gar_bwd_ms", "t_olp_moe_bwd_ms")
    cast = {"r_fwd": int, "case_fwd": int, "r_bwd": int, "case_bwd": int,
            "boundary_fwd": bool, "boundary_bwd": bool}
    return {k: cast.get(k, float)(p[k]) for k in keys}


def partition_to_json(out, n_layers: int) -> dict:
    """out: plan.build_partition_plan's flat array."""
    rows = np.asarray(out[: 9 * n_layers]).reshape(n_layers, 9)
    layers = [{"n_first": float(r[0]), "n_first_dense": float(r[1]), "n_first_moe": float(r[2]),
               "x_g": float(r[3]), "t_gar_ms": float(r[4]),
               "window": {"degree": int(r[5]), "case_id": int(r[6]),
                          "t_olp_moe_ms": float(r[7]), "t_olp_dense_ms": float(r[8])}}
              for r in rows]
    b = 9 * n_layers
    return {"layers": layers, "tail_elements": float(out[b]), "tail_ms": float(out[b + 1]),
            "objective_ms": float(out[b + 2]), "step2_ran": bool(out[b + 3])}


def volumes_to_json(v) -> dict:
    keys = ("a2a_elements", "ag_elements", "rs_elements", "gemm_macs", "gemm_count",
            "grad_elements", "capacity")
    return {k: (int(x) if k in ("gemm_count", "capacity") else float(x)) for k, x in zip(keys, v)}


# --- bench CSV (json_io.cpp:251-307) ---------------------------------------

# std::from_chars(double) general format: optional '-', decimal or
# inf/infinity/nan(...) — no '+', no whitespace, no hex prefix.
_FROM_CHARS = re.compile(r"-?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|inf(?:inity)?|nan(?:\([A-Za-z0-9_]*\))?)",
                         re.IGNORECASE)


def _csv_number(cell, line, what):
    if not _FROM_CHARS.fullmatch(cell):
        raise _err(f"bench csv line {line}: bad {what} '{cell}'")
    return float(cell)


def parse_bench_csv(text: str):
    """(kind, n, t_ms) rows with the reference's line rules: '\\r' stripped,
    empty lines skipped, physical line 1 (when non-empty) must be the header."""
    out, line_no = [], 0
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()                     # getline does not yield the empty tail
    for raw in lines:
        line_no += 1
        line = raw[:-1] if raw.endswith("\r") else raw
        if not line:
            continue
        cells = line.split(",")
        if line_no == 1:
            if cells != ["kind", "n", "t_ms"]:
                raise _err("bench csv line 1: expected header kind,n,t_ms")
            continue
        if len(cells) != 3:
            raise _err(f"bench csv line {line_no}: expected 3 fields, got {len(cells)}")
        if cells[0] not in KIND_ORDER:
            raise _err(f"bench csv line {line_no}: unknown kind '{cells[0]}'")
        out.append((cells[0], _csv_number(cells[1], line_no, "n"),
                    _csv_number(cells[2], line_no, "t_ms")))
    if line_no == 0:
        raise _err("bench csv line 1: empty file")
    return out


def load_bench_csv(path):
    return parse_bench_csv(read_text_file(path))


def format_double(v: float) -> str:
    """std::to_chars(double) shortest form: the shortest round-trip digits in
    fixed or scientific notation, whichever is shorter (fixed on a tie),
    exponent with at least two digits, an integral fixed value printed exactly
    (json_io.cpp:322-326)."""
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    a = abs(v)
    if a == 0.0:
        return sign + "0"
    digits, exp = _shortest_digits(a)         # a = 0.d1d2... x 10^exp
    sci_m = digits[0] + ("." + digits[1:] if len(digits) > 1 else "")
    e = exp - 1
    sci = f"{sci_m}e{'-' if e < 0 else '+'}{abs(e):02d}"
    if exp <= 0:
        fixed = "0." + "0" * (-exp) + digits
    elif exp >= len(digits):
        fixed = str(int(a))    # to_chars prints an integral value's exact digits

    else:
        fixed = digits[:exp] + "." + digits[exp:]
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def _shortest_digits(a: float):
    r = repr(a)                                # shortest round-trip (Python >= 3.1)
    m, _, e = r.partition("e")
    exp = int(e) if e else 0
    ip, _, fp = m.partition(".")
    if fp == "0":
        fp = ""
    digits = (ip + fp).lstrip("0")
    lead = len(ip) if ip != "0" else -(len(fp) - len(fp.lstrip("0")))
    digits = digits.rstrip("0") or "0"
    return digits, exp + lead


# --- the planner subcommands (main.cpp:79-291) -----------------------------

def _env_int(name):
    raw = os.environ.get(name)
    if raw is None:
        return -1
    if not re.fullmatch(r"-?\d+", raw) or int(raw) < 1 or int(raw) > 2**31 - 1:
        raise _err(f"{name}: invalid value '{raw}'")
    return int(raw)


def _env_seed():
    raw = os.environ.get("FSMOE_SEED")
    if raw is None:
        return None
    if not re.fullmatch(r"\d+", raw) or int(raw) >= 2**64:
        raise _err(f"FSMOE_SEED: invalid value '{raw}'")
    return int(raw)


def resolve_r_max(flag_value: int, file_value: int) -> int:
    """Flag > FSMOE_R_MAX > config file (main.cpp:48-54)."""
    if flag_value > 0:
        return flag_value
    env = _env_int("FSMOE_R_MAX")
    return env if env > 0 else file_value


def cmd_fit(bench_path, min_r2=0.99):
    prof, worst, mask = P.fit_profile(load_bench_csv(bench_path), min_r2)
    doc = profile_to_json(prof)
    doc["fit"] = {"min_r_squared": float(worst),
                  "clamped_kinds": [k for i, k in enumerate(KIND_ORDER) if mask >> i & 1]}
    return doc


def plan_model(model_path, profile_path, r_max_flag=0, seed_flag=None):
    """main.cpp:103-130: volumes per layer, build_partition_plan, then each
    layer's plan_layer under its partition's t_gar."""
    m = load_model(model_path)
    prof = load_profile(profile_path)
    r_max = resolve_r_max(r_max_flag, m["r_max"])
    de = list(m["de"])
    env_seed = _env_seed()
    if env_seed is not None:
        de[4] = env_seed
    if seed_flag is not None:
        de[4] = seed_flag
    vols = [P.derive_volumes(l, m["parallel"]) for l in m["layers"]]
    part = P.build_partition_plan([(v, l.t_olp_dense_ms, float(v[5])) for v, l in zip(vols, m["layers"])],
                                  prof, tuple(de), r_max=r_max)
    n = len(vols)
    t_gar = np.asarray(part[: 9 * n]).reshape(n, 9)[:, 4]
    pipes = [P.plan_layer(v, prof, t_gar_bwd_ms=float(t), r_max=r_max) for v, t in zip(vols, t_gar)]
    return {"r_max": r_max, "seed": int(de[4]),
            "layers": [{"index": i, "volumes": volumes_to_json(v), "pipeline": plan_to_json(p)}
                       for i, (v, p) in enumerate(zip(vols, pipes))],
            "partition": partition_to_json(part, n)}


def cmd_simulate(model_path, profile_path, style="fsmoe", pass_="fwd", layer_index=0,
                 r_max_flag=0):
    """main.cpp:155-210 (report only; the trace / timeline writers stay in
    the reference's CLI)."""
    if style not in P.STYLES:
        raise _err(f"unknown schedule style '{style}'")
    if pass_ not in ("fwd", "bwd"):
        raise _err("simulate: pass must be fwd or bwd")
    m = load_model(model_path)
    prof = load_profile(profile_path)
    r_max = resolve_r_max(r_max_flag, m["r_max"])
    if layer_index < 0 or layer_index >= len(m["layers"]):
        raise _err("simulate: layer index out of range")
    vol = P.derive_volumes(m["layers"][layer_index], m["parallel"])
    t_gar = 0.0
    if pass_ == "bwd" and vol[5] > 0:
        t_gar = prof[6] + vol[5] * prof[7]      # predict_ms(profile.ar, grad), cost_models.cpp:9-11
    plan = P.plan_layer(vol, prof, t_gar_bwd_ms=t_gar, r_max=r_max)
    r = plan["r_fwd"] if pass_ == "fwd" else plan["r_bwd"]
    out = P.simulate_stage(vol, prof, 1 if pass_ == "fwd" else 2, r,
                           sync_ms=[t_gar] if t_gar > 0 else (), style=style)
    mk = float(out[0])
    busy = {res: float(out[1 + i]) for i, res in enumerate(RESOURCES)}
    return {"style": style, "pass": pass_, "layer": layer_index, "r": int(r), "makespan_ms": mk,
            "busy_ms": busy, "utilization": {k: (b / mk if mk > 0 else 0.0) for k, b in busy.items()}}


def json_close(a, b, tol: float) -> bool:
    """main.cpp:239-264: numbers within tol * max(1, |x|, |y|), same shape."""
    num = (int, float)
    if isinstance(a, num) and not isinstance(a, bool) and isinstance(b, num) and not isinstance(b, bool):
        x, y = float(a), float(b)
        return abs(x - y) <= tol * max(1.0, abs(x), abs(y))
    if type(a) is not type(b):
        return False
    if isinstance(a, dict):
        return len(a) == len(b) and all(k in b and json_close(v, b[k], tol) for k, v in a.items())
    if isinstance(a, list):
        return len(a) == len(b) and all(json_close(x, y, tol) for x, y in zip(a, b))
    return a == b


def _emit(path, text):
    if path:
        write_text_file(path, text)
    else:
        sys.stdout.write(text)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="planio", description="MoE training schedule planner and simulator")
    ap.add_argument("--verbose", action="store_true")
    sub = ap.add_subparsers(dest="cmd", required=True)
    f = sub.add_parser("fit")
    f.add_argument("--bench", required=True)
    f.add_argument("--out", default="")
    f.add_argument("--min-r2", type=float, default=0.99)
    p = sub.add_parser("plan")
    p.add_argument("--model", required=True)
    p.add_argument("--profile", required=True)
    p.add_argument("--out", default="")
    p.add_argument("--r-max", type=int, default=0)
    p.add_argument("--seed", type=int, default=None)
    s = sub.add_parser("simulate")
    s.add_argument("--model", required=True)
    s.add_argument("--profile", required=True)
    s.add_argument("--style", default="fsmoe")
    s.add_argument("--pass", dest="pass_", default="fwd")
    s.add_argument("--layer", type=int, default=0)
    s.add_argument("--out", default="")
    s.add_argument("--r-max", type=int, default=0)
    c = sub.add_parser("compare")
    c.add_argument("a")
    c.add_argument("b")
    c.add_argument("--tol", type=float, default=1e-9)
    a = ap.parse_args(argv)
    try:
        if a.cmd == "fit":
            doc = cmd_fit(a.bench, a.min_r2)
            _emit(a.out, dumps(doc))
            sys.stderr.write(f"fit: worst r^2 {doc['fit']['min_r_squared']:.6g}\n")
        elif a.cmd == "plan":
            _emit(a.out, dumps(plan_model(a.model, a.profile, a.r_max, a.seed)))
        elif a.cmd == "simulate":
            _emit(a.out, dumps(cmd_simulate(a.model, a.profile, a.style, a.pass_, a.layer, a.r_max)))
        else:
            try:
                ja = json.loads(read_text_file(a.a))
                jb = json.loads(read_text_file(a.b))
            except json.JSONDecodeError as e:
                raise _err(f"compare: {e}") from None
            if json_close(ja, jb, a.tol):
                print(f"equal within tolerance {a.tol:g}")
                return 0
            print(f"documents differ beyond tolerance {a.tol:g}")
            return 1
    except NL.ConfigError as e:
        sys.stderr.write(f"error: {e}\n")
        return 2
    except NL.FitQualityError as e:
        sys.stderr.write(f"error: {e}\n")
        return 3
    except NL.InvariantError as e:
        sys.stderr.write(f"internal error: {e}\n")
        return 4
    return 0


if __name__ == "__main__":
    sys.exit(main())
