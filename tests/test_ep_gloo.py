"""Expert-parallel protocol of the executor (paper_2501_10714_b200/cpp/
moe_layer.cpp), run on CPU with world_size 2 over gloo: each rank routes its
own tokens with local capacity C, ships rows [lo, hi) of every (rank, expert)
block per pipeline chunk (the executor's 128-row granule chunks, fetched from
libfsmoe.so), runs its local experts, ships the results back and combines.
Forward outputs and backward gradients must equal the single-device fp64
restatement applied per rank with the union of experts (expert grads summed
over ranks, replicated gate grads allreduced) — the EP semantics of SURVEY.md
§8(e). Also checks the NCCL unique-id bootstrap broadcast. CPU only."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(send, recv, chunks, P, El, C, M):
    """send/recv: [P*El, C, M]; per chunk pack rows [lo,hi) per peer, all_to_all."""
    for lo, hi in chunks:
        n = hi - lo
        buf = torch.from_numpy(np.ascontiguousarray(send.reshape(P, El, C, M)[:, :, lo:hi, :]))
        out = torch.empty_like(buf)
        dist.all_to_all_single(out.view(-1), buf.view(-1))
        recv.reshape(P, El, C, M)[:, :, lo:hi, :] = out.numpy()
        assert n > 0


def _worker(rank, world, port, r, ffn, result_q):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import layer_oracle
    import pyoracle
    from paper_2501_10714_b200 import plan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        T, M, H, E, k = 96, 16, 128 if ffn == "simple" else 128, 4, 2
        P, El = world, E // world
        C = 40 if r == 1 else 320  # tight (drops) / roomy with 3 granule chunks
        rng = np.random.default_rng(0)
        wg = rng.uniform(-1, 1, (M, E)) / 4
        wn = rng.uniform(-1, 1, (M, E)) / 4
        N1 = H if ffn == "simple" else 2 * H
        W1 = rng.uniform(-1, 1, (E, N1, M)) / 4
        W2 = rng.uniform(-1, 1, (E, M, H)) / 8
        xr = np.random.default_rng(100 + rank)
        x = xr.uniform(-1, 1, (T, M))
        dy = xr.uniform(-1, 1, (T, M))
        orc = pyoracle.Oracle("port")

        # ---- single-device restatement on this rank's tokens (the contract)
        y_ref, cache = layer_oracle.forward(x, "noisy_topk", k, 5, C, wg, wn, None, W1, W2, ffn, orc)
        g_ref = layer_oracle.backward(cache, dy, "noisy_topk", k, C, wg, wn, None, W1, W2, ffn)

        # ---- the executor's EP protocol
        g = orc.run_gate("noisy_topk", k, 5, x, wg, wn)
        d = orc.dispatch(x, E, g.token, g.expert, C)
        fill = torch.from_numpy(d.fill.copy())
        rfill = torch.empty_like(fill)
        dist.all_to_all_single(rfill, fill)  # E_l counts per peer (rank-major)
        chunks = plan.pipeline_chunks(C, r)
        assert len(chunks) == r
        Xs = d.buffers.reshape(E, C, M)
        Xr = np.zeros_like(Xs)
        _exchange(Xs, Xr, chunks, P, El, C, M)
        Or = np.zeros_like(Xr)
        Z, Hh = {}, {}
        for b in range(P * El):  # recv block (src p, local expert el)
            e = rank * El + b % El
            Z[b] = Xr[b] @ W1[e].T
            if ffn == "gated3":
                gt, u = layer_oracle.split_gated(Z[b], H)
                Hh[b] = gt * layer_oracle.sigmoid(gt) * u
            else:
                Hh[b] = layer_oracle.gelu(Z[b])
            Or[b] = Hh[b] @ W2[e].T
        Os = np.zeros_like(Or)
        _exchange(Or, Os, chunks, P, El, C, M)
        y = orc.combine(Os.reshape(E * C, M), T, E, g.token, g.expert, g.weight, d.slot_of_pick, M)
        assert np.abs(y - y_ref).max() <= 1e-12 * max(1.0, np.abs(y_ref).max())
        # padding rows never carry data past the exchanged fill counts
        assert all(int(rfill[b]) <= C for b in range(P * El))

        # backward: dO on the send side, exchange, expert dgrad/wgrad, back
        dO = np.zeros((E * C, M))
        dw = np.zeros(g.token.size)
        for p in range(g.token.size):
            s = d.slot_of_pick[p]
            if s >= 0:
                dO[s] = g.weight[p] * dy[g.token[p]]
                dw[p] = dy[g.token[p]] @ Os.reshape(E * C, M)[s]
        dOr = np.zeros_like(Xr)
        _exchange(dO.reshape(E, C, M), dOr, chunks, P, El, C, M)
        gW1 = np.zeros((El, N1, M))
        gW2 = np.zeros((El, M, H))
        dXr = np.zeros_like(Xr)
        for b in range(P * El):
            el = b % El
            e = rank * El + el
            dH = dOr[b] @ W2[e]
            gW2[el] += dOr[b].T @ Hh[b]
            if ffn == "gated3":
                gt, u = layer_oracle.split_gated(Z[b], H)
                sg = layer_oracle.sigmoid(gt)
                dZ = layer_oracle.join_gated(dH * u * sg * (1 + gt * (1 - sg)), dH * gt * sg)
            else:
                dZ = dH * layer_oracle.gelu_grad(Z[b])
            gW1[el] += dZ.T @ Xr[b]
            dXr[b] = dZ @ W1[e]
        dXs = np.zeros_like(dXr)
        _exchange(dXr, dXs, chunks, P, El, C, M)
        dx = np.zeros((T, M))
        for p in range(g.token.size):
            s = d.slot_of_pick[p]
            if s >= 0:
                dx[g.token[p]] += dXs.reshape(E * C, M)[s]
        tol = 1e-10
        # expert grads: the owner's gradient is the sum of every rank's contribution
        contrib = torch.from_numpy(np.ascontiguousarray(g_ref["g_w1"]))
        dist.all_reduce(contrib)
        want_w1 = contrib.numpy()[rank * El:(rank + 1) * El]
        contrib2 = torch.from_numpy(np.ascontiguousarray(g_ref["g_w2"]))
        dist.all_reduce(contrib2)
        want_w2 = contrib2.numpy()[rank * El:(rank + 1) * El]
        assert np.abs(gW1 - want_w1).max() <= tol * max(1.0, np.abs(want_w1).max())
        assert np.abs(gW2 - want_w2).max() <= tol * max(1.0, np.abs(want_w2).max())
        # token gradient: expert path equals the restatement's (gate path is local)
        dx_expert_ref = g_ref["dx"] - _gate_dx(layer_oracle, cache, dy, g_ref, x, wg, wn, k)
        assert np.abs(dx - dx_expert_ref).max() <= tol * max(1.0, np.abs(dx_expert_ref).max())
        # replicated gate parameters: gradients allreduced over the EP group
        gg = torch.from_numpy(np.ascontiguousarray(g_ref["g_gate"]))
        dist.all_reduce(gg)
        result_q.put((rank, "ok", float(np.abs(gg.numpy()).max())))
    except Exception as e:  # surface the failure to the parent
        result_q.put((rank, f"error: {e!r}", 0.0))
        raise
    finally:
        dist.destroy_process_group()


def _gate_dx(layer_oracle, cache, dy, g_ref, x, wg, wn, k):
    """dx contribution of the gate alone (restatement minus the expert path)."""
    T, M = x.shape
    g, d = cache.picks, cache.disp
    E = wg.shape[1]
    dw = np.zeros(g.token.size)
    O2 = cache.O.reshape(-1, M)
    for p in range(g.token.size):
        s = d.slot_of_pick[p]
        if s >= 0:
            dw[p] = dy[g.token[p]] @ O2[s]
    dS = np.zeros((T, E))
    for t in range(T):
        sl = slice(t * k, (t + 1) * k)
        ee, ww, dd = g.expert[sl], g.weight[sl], dw[sl]
        dS[t, ee] = ww * (dd - np.sum(ww * dd))
    dZn = dS * cache.noise * layer_oracle.sigmoid(cache.spread)
    return dS @ wg.T + dZn @ wn.T


@pytest.mark.parametrize("r", [1, 3])
@pytest.mark.parametrize("ffn", ["simple", "gated3"])
def test_ep_protocol_world2_matches_single_device(r, ffn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(i, 2, port, r, ffn, q)) for i in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(s == "ok" for _, s, _ in res), res


def _uid_worker(rank, world, port, q):
    sys.path[:0] = [ROOT]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2501_10714_b200.layer import broadcast_unique_id
    uid = bytes(range(128)) if rank == 0 else bytes(128)
    got = broadcast_unique_id(uid, world)
    q.put((rank, got == bytes(range(128))))
    dist.destroy_process_group()


def test_nccl_unique_id_bootstrap_broadcast():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_uid_worker, args=(i, 2, port, q)) for i in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=30)
    assert all(ok for _, ok in res), res
