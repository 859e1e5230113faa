"""Expert parallelism: routed experts sharded across ranks, tokens dispatched
and combined with all-to-all.

Partition: contiguous expert blocks, uneven when E % G != 0 (Qwen 60 over 8
ranks -> 8,8,8,8,7,7,7,7).  Router, shared experts, attention and the head
are replicated; every token is routed, gated and combined on its HOME rank,
so routing / fallback decisions do not depend on G.  One layer:

  1. home: router + top-k (+ replay)                    (libmobile router)
  2. home: pairs sorted by owner rank (stable), counts all-to-all, then the
     pair rows (h2 row of the token) + owner-local expert ids all-to-all
  3. owner: expert FFN on the received rows             (libmobile kernels)
  4. owner -> home: all-to-all of the output rows back in the same order
  5. home: un-permute to pair order, combine in SELECTION order + shared
     experts + residual                                 (libmobile combine)

Every expert output row is a fixed-order dot product independent of which
other rows share its launch, and the combine order is fixed on the home rank,
so the layer output is bit-identical for G = 1, 2, 4, 8.

The exchange is written against torch.distributed (NCCL over NVLink on the
B200 box, gloo in the CPU tests); the expert compute is a callable so the
host-side exchange logic can be tested on CPU with the oracle as the expert.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def partition(E: int, G: int) -> list[tuple[int, int]]:
    """Contiguous expert blocks [lo, hi) per rank, the first E % G ranks one larger."""
    base, extra = divmod(E, G)
    out, lo = [], 0
    for r in range(G):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def owner_table(E: int, G: int, device) -> tuple[torch.Tensor, torch.Tensor]:
    """(owner rank of each expert, expert index local to its owner)."""
    own = torch.empty(E, dtype=torch.long)
    loc = torch.empty(E, dtype=torch.long)
    for r, (lo, hi) in enumerate(partition(E, G)):
        own[lo:hi] = r
        loc[lo:hi] = torch.arange(hi - lo)
    return own.to(device), loc.to(device)


@dataclass
class DispatchPlan:
    order: torch.Tensor  # (P_valid,) pair ids sorted by (owner rank, pair id)
    send_counts: list[int]
    recv_counts: list[int]


class EPExchange:
    """Token dispatch / combine for one expert-parallel group."""

    def __init__(self, E: int, group=None):
        self.group = group
        self.G = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.E = E
        self.parts = partition(E, self.G)

    def _a2a(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits):
        if self.G == 1:
            out.copy_(inp)
            return out
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)
        return out

    def plan(self, idx: torch.Tensor, k_tok: torch.Tensor) -> DispatchPlan:
        """idx (T, k_max) selections of this rank's tokens -> stable send order."""
        T, k_max = idx.shape
        dev = idx.device
        own, _ = owner_table(self.E, self.G, dev)
        slot = torch.arange(k_max, device=dev)[None, :].expand(T, k_max)
        valid = (slot < k_tok[:, None].long()) & (idx >= 0)
        pair = torch.arange(T * k_max, device=dev).reshape(T, k_max)[valid]
        e = idx.long()[valid]
        dest = own[e]
        # stable sort by destination: key = dest * P + pair
        key = dest * (T * k_max + 1) + pair
        order = pair[torch.argsort(key)]
        send = torch.bincount(dest, minlength=self.G).to(torch.long)
        recv = torch.empty_like(send)
        self._a2a(recv, send, [1] * self.G, [1] * self.G)
        return DispatchPlan(order, send.cpu().tolist(), recv.cpu().tolist())

    def dispatch(self, plan: DispatchPlan, rows_by_pair: torch.Tensor, idx: torch.Tensor):
        """Send each pair's activation row + owner-local expert id to the owner.
        Returns (received rows (R, d), received local expert ids (R,))."""
        k_max = idx.shape[1]
        dev = rows_by_pair.device
        _, loc = owner_table(self.E, self.G, dev)
        send_rows = rows_by_pair[plan.order // k_max].contiguous()
        send_ids = loc[idx.reshape(-1).long()[plan.order]].contiguous()
        R = sum(plan.recv_counts)
        recv_rows = torch.empty(R, rows_by_pair.shape[1], dtype=rows_by_pair.dtype, device=dev)
        recv_ids = torch.empty(R, dtype=send_ids.dtype, device=dev)
        self._a2a(recv_rows, send_rows, plan.recv_counts, plan.send_counts)
        self._a2a(recv_ids, send_ids, plan.recv_counts, plan.send_counts)
        return recv_rows, recv_ids

    def combine(self, plan: DispatchPlan, out_rows: torch.Tensor, T: int, k_max: int) -> torch.Tensor:
        """Return the owners' output rows to their home pairs: Y (T*k_max, d),
        rows of unselected slots left zero."""
        S = sum(plan.send_counts)
        back = torch.empty(S, out_rows.shape[1], dtype=out_rows.dtype, device=out_rows.device)
        self._a2a(back, out_rows.contiguous(), plan.send_counts, plan.recv_counts)
        Y = torch.zeros(T * k_max, out_rows.shape[1], dtype=out_rows.dtype, device=out_rows.device)
        Y[plan.order] = back
        return Y


class ExpertParallelMoE:
    """MoBiLE MoE layer with expert-parallel routed experts on the device.

    `local` is a MoBiLEMoE over DeviceWeights holding only this rank's routed
    experts (router, shared experts replicated).  Decisions, gates and the
    combine run on the home rank with the same libmobile kernels as the
    single-GPU layer; only the routed expert rows travel.
    """

    def __init__(self, moe_full_router, local_moe, E: int, group=None):
        self.router_moe = moe_full_router  # MoBiLEMoE (router + shared weights)
        self.local = local_moe             # MoBiLEMoE with the local expert block
        self.x = EPExchange(E, group)

    def forward(self, x, layer, k_tok, k_max, replay=None, replay_mask=None, reuse_gates=False, ln_out=None):
        from . import kernels as K
        T = x.shape[0]
        rm = self.router_moe
        sc = rm.route(x, layer, k_tok, k_max, replay=replay, replay_mask=replay_mask, reuse_gates=reuse_gates)
        r = sc["router"]
        plan = self.x.plan(r["idx"], k_tok)
        rows, ids = self.x.dispatch(plan, r["h2"], r["idx"])
        out = self.local_expert_rows(layer, rows, ids)
        Y = self.x.combine(plan, out, T, k_max)
        Ys = None
        if rm.S:
            Ys = rm.shared_rows(layer, r["h2"], sc)
        shared_logits = r["extra"] if rm.dw.n_gate_rows else None
        return K.combine(x, Y, r["gates"], k_tok, Ys, rm.S, shared_logits, ln_out=ln_out)

    def local_expert_rows(self, layer, rows: torch.Tensor, ids: torch.Tensor) -> torch.Tensor:
        """Expert FFN of each received row with its owner-local expert (k = 1)."""
        R = rows.shape[0]
        if R == 0:
            return torch.zeros(0, rows.shape[1], dtype=torch.float32, device=rows.device)
        return self.local.rows_ffn(layer, rows.float().contiguous(), ids.int().contiguous())
