"""TEST INFRASTRUCTURE ONLY — fp64 numpy restatement of the full MoE layer.

Routing (gate -> dispatch -> combine) is the C restatement of the reference
(oracle/fsmoe_oracle.c, pinned to the reference's golden vectors). The expert
FFN, the backward pass and the expert-parallel semantics are ABSENT from the
reference (workload.cpp:70 only counts GEMMs): for those this
module is the builder-defined contract of SURVEY.md Appendix D, so their
parity is "unpinned by the reference" and checked here against this fp64
restatement with stated tolerances.

FFN kinds:  simple = W2 . gelu_erf(W1 x)        (2 GEMMs)
            gated3 = W2 . (silu(Wg x) * (Wu x))  (3 GEMMs; W1 stores Wg/Wu
                     interleaved in 128-unit blocks: rows [256b, 256b+128) are
                     gate units 128b.., rows [256b+128, 256b+256) up units)
Expert parallelism: each rank routes its own tokens with local capacity C;
expert e lives on rank e // E_local; outputs equal the single-device layer
applied per rank with the union of experts; expert grads sum over ranks,
replicated (gate) grads sum over ranks.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
from scipy.special import erf

try:
    from . import pyoracle
except ImportError:
    import pyoracle


def gelu(z):
    return 0.5 * z * (1.0 + erf(z / np.sqrt(2.0)))


def gelu_grad(z):
    return 0.5 * (1.0 + erf(z / np.sqrt(2.0))) + z * np.exp(-0.5 * z * z) / np.sqrt(2.0 * np.pi)


def sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def split_gated(Z, H):
    """Interleaved [gate128 | up128] columns -> (gate, up), each rows x H."""
    r = Z.shape[0]
    zb = Z.reshape(r, H // 128, 2, 128)
    return zb[:, :, 0, :].reshape(r, H), zb[:, :, 1, :].reshape(r, H)


def join_gated(G, U):
    r, H = G.shape
    out = np.empty((r, H // 128, 2, 128))
    out[:, :, 0, :] = G.reshape(r, H // 128, 128)
    out[:, :, 1, :] = U.reshape(r, H // 128, 128)
    return out.reshape(r, 2 * H)


@dataclass
class Cache:
    x: np.ndarray
    picks: object
    disp: object
    X: np.ndarray
    Z: list
    Hh: list
    O: np.ndarray
    noise: np.ndarray | None
    spread: np.ndarray | None
    scores: np.ndarray | None
    q: np.ndarray | None


def noise_matrix(seed, T, E):
    lib = C.CDLL(pyoracle.PORT_SO)
    lib.orc_noise_row.argtypes = [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_double)]
    out = np.empty((T, E))
    for t in range(T):
        row = out[t]
        lib.orc_noise_row(C.c_uint64(seed), t, E, row.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def forward(x, gate, k, seed, capacity, w_gate, w_noise, proj, W1, W2, ffn, orc=None):
    """x: T x M fp64 (already rounded to the device dtype); W1: [E][N1][M];
    W2: [E][M][H]. Returns (y, cache)."""
    orc = orc or pyoracle.Oracle("port")
    T, M = x.shape
    E = W1.shape[0]
    H = W2.shape[2]
    g = orc.run_gate(gate, k, seed, x, w_gate, w_noise if gate == "noisy_topk" else None,
                     proj if gate == "cosine_topk" else None)
    d = orc.dispatch(x, E, g.token, g.expert, capacity)
    X = d.buffers.reshape(E, capacity, M)
    O = np.zeros_like(X)
    Zs, Hs = [], []
    for e in range(E):
        Z = X[e] @ W1[e].T
        if ffn == "gated3":
            Gt, U = split_gated(Z, H)
            Hh = Gt * sigmoid(Gt) * U
        else:
            Hh = gelu(Z)
        O[e] = Hh @ W2[e].T
        Zs.append(Z)
        Hs.append(Hh)
    y = orc.combine(O.reshape(E * capacity, M), T, E, g.token, g.expert, g.weight,
                    d.slot_of_pick, M)
    noise = spread = scores = q = None
    if gate == "noisy_topk":
        noise = noise_matrix(seed, T, E)
        spread = x @ w_noise
        scores = x @ w_gate + noise * np.log1p(np.exp(spread))
    elif gate == "sigmoid_topk":
        scores = x @ w_gate
    elif gate == "expert_choice":
        scores = x @ w_gate
    elif gate == "cosine_topk":
        q = x @ proj.T
        qn = np.linalg.norm(q, axis=1, keepdims=True)
        wn = np.linalg.norm(w_gate, axis=0, keepdims=True)
        scores = (q @ w_gate) / (qn * wn)
    return y, Cache(x, g, d, X, Zs, Hs, O, noise, spread, scores, q)


def backward(cache, dy, gate, k, capacity, w_gate, w_noise, proj, W1, W2, ffn):
    """Returns dict(dx, g_gate, g_noise, g_proj, g_w1, g_w2) in fp64."""
    x, g, d = cache.x, cache.picks, cache.disp
    T, M = x.shape
    E = W1.shape[0]
    H = W2.shape[2]
    P = g.token.size
    # combine backward
    dO = np.zeros((E * capacity, M))
    dw = np.zeros(P)
    O2 = cache.O.reshape(E * capacity, M)
    for p in range(P):
        s = d.slot_of_pick[p]
        if s >= 0:
            dO[s] = g.weight[p] * dy[g.token[p]]
            dw[p] = dy[g.token[p]] @ O2[s]
    dO = dO.reshape(E, capacity, M)
    g_w1 = np.zeros_like(W1)
    g_w2 = np.zeros_like(W2)
    dX = np.zeros_like(cache.X)
    for e in range(E):
        dHh = dO[e] @ W2[e]
        g_w2[e] = dO[e].T @ cache.Hh[e]
        Z = cache.Z[e]
        if ffn == "gated3":
            Gt, U = split_gated(Z, H)
            sg = sigmoid(Gt)
            dG = dHh * U * sg * (1.0 + Gt * (1.0 - sg))
            dU = dHh * Gt * sg
            dZ = join_gated(dG, dU)
        else:
            dZ = dHh * gelu_grad(Z)
        g_w1[e] = dZ.T @ cache.X[e]
        dX[e] = dZ @ W1[e]
    dXf = dX.reshape(E * capacity, M)
    dx = np.zeros((T, M))
    for p in range(P):
        s = d.slot_of_pick[p]
        if s >= 0:
            dx[g.token[p]] += dXf[s]
    # gate backward
    g_gate = np.zeros_like(w_gate)
    g_noise = np.zeros_like(w_noise) if w_noise is not None else None
    g_proj = np.zeros_like(proj) if proj is not None else None
    if gate == "expert_choice":
        dS = np.zeros((T, E))
        Ck = P // E
        for e in range(E):
            sl = slice(e * Ck, (e + 1) * Ck)
            sig = np.sum(g.weight[sl] * dw[sl])
            dS[g.token[sl], e] = g.weight[sl] * (dw[sl] - sig)
        g_gate += x.T @ dS
        dx += dS @ w_gate.T
    else:
        dS = np.zeros((T, E))
        for t in range(T):
            sl = slice(t * k, (t + 1) * k)
            ee, ww, dd = g.expert[sl], g.weight[sl], dw[sl]
            if gate == "sigmoid_topk":
                dS[t, ee] = dd * ww * (1.0 - ww)
            else:
                dS[t, ee] = ww * (dd - np.sum(ww * dd))
        if gate == "cosine_topk":
            q = cache.q
            qn = np.linalg.norm(q, axis=1, keepdims=True)
            wn = np.linalg.norm(w_gate, axis=0, keepdims=True)
            s = cache.scores
            # ds/dq and ds/dw (Appendix D)
            dq = (dS / (qn * wn)) @ w_gate.T - (np.sum(dS * s, axis=1, keepdims=True)) * q / qn ** 2
            g_gate += (q / qn).T @ dS / wn - w_gate * np.sum(dS * s, axis=0, keepdims=True) / wn ** 2
            g_proj += dq.T @ x
            dx += dq @ proj
        else:
            g_gate += x.T @ dS
            dx += dS @ w_gate.T
            if gate == "noisy_topk":
                dZn = dS * cache.noise * sigmoid(cache.spread)
                g_noise += x.T @ dZn
                dx += dZn @ w_noise.T
    return dict(dx=dx, g_gate=g_gate, g_noise=g_noise, g_proj=g_proj, g_w1=g_w1, g_w2=g_w2)
