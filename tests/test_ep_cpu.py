"""Expert-parallel dispatch/combine (ep.py) with world_size 2 over gloo on CPU.

The expert compute is the oracle (the exchange logic is what is under test);
the expert-parallel layer output must be bit-identical to the single-rank
oracle layer for every rank's tokens (decisions on the home rank, fixed
combine order), including uneven expert partitions and ragged per-token widths.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import moe_ref as R

SPEC = dict(num_layers=1, num_experts=7, k_big=3, k_little=1, hidden_dim=16, vocab_size=32, seed=4, ffn_dim=8,
            activation="swiglu", n_shared=1, shared_ffn_dim=8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tokens(rank):
    rng = np.random.default_rng(100 + rank)
    T = 5 + rank  # ragged batch per rank
    h2 = rng.normal(size=(T, SPEC["hidden_dim"]))
    k_tok = rng.integers(1, SPEC["k_big"] + 1, size=T)
    return h2, k_tok


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_12357_b200.ep import EPExchange, partition
        W = R.build_weights(R.OracleSpec(**SPEC))
        E, k_max = SPEC["num_experts"], SPEC["k_big"]
        h2, k_tok = _tokens(rank)
        T = h2.shape[0]
        logits = h2 @ W.router[0]
        sels = [R.route_token(logits[t], int(k_tok[t]))[0] for t in range(T)]
        gates = [R.route_token(logits[t], int(k_tok[t]))[1] for t in range(T)]
        idx = torch.full((T, k_max), -1, dtype=torch.long)
        for t, sel in enumerate(sels):
            idx[t, :len(sel)] = torch.tensor(sel)
        ex = EPExchange(E)
        plan = ex.plan(idx, torch.tensor(k_tok))
        rows, ids = ex.dispatch(plan, torch.tensor(h2), idx)
        lo, hi = partition(E, world)[rank]
        out = torch.zeros(rows.shape[0], SPEC["hidden_dim"], dtype=torch.float64)
        for i in range(rows.shape[0]):  # owner: oracle expert FFN on each received row
            e = lo + int(ids[i])
            assert lo <= e < hi
            out[i] = torch.from_numpy(R._expert(rows[i].numpy(), W.expert_in[0, e], W.expert_up[0, e],
                                                W.expert_out[0, e], "swiglu"))
        Y = ex.combine(plan, out, T, k_max).numpy()
        # home combine in selection order + shared expert (toymoe.py:204, 207 order)
        moe = np.zeros_like(h2)
        for t in range(T):
            for j, g in enumerate(gates[t]):
                moe[t] += g * Y[t * k_max + j]
        moe += R._expert(h2, W.shared_in[0, 0], W.shared_up[0, 0], W.shared_out[0, 0], "swiglu")
        ref = R.moe_block(W, 0, h2, k_tok)
        q.put((rank, bool(np.array_equal(moe, ref.out)), float(np.abs(moe - ref.out).max()),
               plan.send_counts, plan.recv_counts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ep_exchange_bit_identical(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, err, send, recv in res:
        assert same, (rank, err)
    # every pair sent is received exactly once somewhere
    assert sum(sum(s) for _, _, _, s, _ in res) == sum(sum(r) for _, _, _, _, r in res)


def test_partition_uneven():
    from paper_2510_12357_b200.ep import partition
    assert [hi - lo for lo, hi in partition(60, 8)] == [8, 8, 8, 8, 7, 7, 7, 7]
    assert partition(8, 8) == [(i, i + 1) for i in range(8)]
    assert partition(64, 1) == [(0, 64)]
