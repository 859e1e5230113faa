"""Expert parallelism over peer memory (csrc/ep_p2p.cu): dispatch / combine by
direct stores into IPC-mapped mailboxes with system-scope flags.

world size 1 in-process, and world size 2 as two processes sharing the one
GPU of a gpurun box (CUDA IPC maps each process's mailbox into the other;
on an NVSwitch node the same stores travel over NVLink).  The reference is
the single-GPU MoBiLE layer on the same tokens: the owner runs its experts
on its mailbox rows with the tcgen05 grouped GEMM (bf16 activations), so the
bar is the bf16 one (2e-2 of the largest output)."""
import os
import socket

import numpy as np
import pytest
import torch

from tests.helpers import QWEN_MINI, matched

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tokens(ms, rank, T):
    rng = np.random.default_rng(1000 + rank)
    x = torch.tensor(rng.normal(size=(T, ms.hidden_dim)), dtype=torch.float32, device="cuda")
    k_tok = torch.tensor(rng.choice([ms.k_little, ms.k_big], size=T), dtype=torch.int32, device="cuda")
    return x, k_tok


def _run(rank, world, T, layers=2):
    """Layer outputs of the P2P EP layer and of the single-GPU layer for this rank's tokens."""
    from paper_2510_12357_b200.ep import P2PExpertParallelMoE, partition
    from paper_2510_12357_b200.model import MoBiLEMoE
    o, ms, dm = matched(QWEN_MINI, "bfloat16")
    lo, hi = partition(ms.num_experts, world)[rank]
    local = MoBiLEMoE(dm.dw.shard_experts(lo, hi))
    ep = P2PExpertParallelMoE(dm.moe, local, ms.num_experts, ms.hidden_dim, cap=T * ms.k_big)
    errs = []
    try:
        for layer in range(layers):
            for rep in range(2):  # repeated exchanges reuse the mailboxes (epochs)
                x, k_tok = _tokens(ms, rank * 10 + layer * 2 + rep, T)
                want, _ = dm.moe.forward(x, layer % ms.num_layers, k_tok, ms.k_big)
                want = want.clone()
                got = ep.forward(x, layer % ms.num_layers, k_tok, ms.k_big)
                torch.cuda.synchronize()
                errs.append((got - want).abs().max().item() / want.abs().max().item())
        assert int(ep.x.flags.item()) == 0
    finally:
        ep.x.close()
    return errs


@pytest.mark.parametrize("T", [1, 6, 40])
def test_p2p_ep_world1(cuda_ok, T):
    errs = _run(0, 1, T)
    assert max(errs) < 2e-2, errs


def _worker(rank, world, port, T, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _run(rank, world, T), None))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, None, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T", [3, 24])
def test_p2p_ep_world2_one_gpu(cuda_ok, T):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, T, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for rank, errs, exc in res:
        assert exc is None, (rank, exc)
        assert max(errs) < 2e-2, (rank, errs)


@pytest.mark.parametrize("T,k_max,E,G", [(5, 3, 7, 2), (300, 4, 60, 8), (1, 2, 8, 3), (2048, 2, 8, 8)])
def test_p2p_plan_matches_nccl_path_order(cuda_ok, T, k_max, E, G):
    """ep_plan_kernel: each valid pair's (owner, position) equals the stable
    (owner, pair id) order of EPExchange.plan; unselected slots (-1 ids,
    k_tok < k_max) are skipped; per-owner counts match."""
    import ctypes as C

    from paper_2510_12357_b200 import _native as N
    from paper_2510_12357_b200.ep import owner_table
    rng = np.random.default_rng(T + E)
    idx = np.stack([rng.permutation(E)[:k_max] for _ in range(T)]).astype(np.int32)
    k_tok = rng.integers(1, k_max + 1, size=T).astype(np.int32)
    idx[rng.random((T, k_max)) < 0.05] = -1
    dev = torch.device("cuda")
    own, loc = owner_table(E, G, dev)
    P = T * k_max
    cap = P
    dest = torch.full((P,), -7, dtype=torch.int32, device=dev)
    counts = torch.zeros(G, dtype=torch.int32, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    box = C.c_void_p()
    N.check(N.lib.mobile_ep_mailbox_create(G, cap, 8, C.byref(box)), "mailbox")
    try:
        peers = torch.tensor([box.value] * G, dtype=torch.int64, device=dev)  # every "peer" is this mailbox
        rows = torch.zeros(T, 8, device=dev)
        ti, tk = torch.tensor(idx, device=dev), torch.tensor(k_tok, device=dev)
        own32, loc32 = own.int().contiguous(), loc.int().contiguous()  # alive until the kernels ran
        N.check(N.lib.mobile_ep_dispatch(N.ptr(rows), N.ptr(ti), N.ptr(tk), T, k_max, 8, N.ptr(own32),
                                         N.ptr(loc32), N.ptr(peers), G, 0, cap, 1, None, 0, N.ptr(dest),
                                         N.ptr(counts), N.ptr(flags), torch.cuda.current_stream().cuda_stream), "dispatch")
        torch.cuda.synchronize()
    finally:
        N.lib.mobile_ep_mailbox_destroy(box)
    d = dest.cpu().numpy()
    owner = own.cpu().numpy()
    want_pos, seen = {}, [0] * G
    for p in range(P):
        t, j = divmod(p, k_max)
        e = idx[t, j]
        if j < k_tok[t] and e >= 0:
            g = owner[e]
            want_pos[p] = g * cap + seen[g]
            seen[g] += 1
    for p in range(P):
        assert d[p] == want_pos.get(p, -1), (p, d[p], want_pos.get(p, -1))
    assert counts.cpu().tolist() == seen
    assert int(flags.item()) == 0
