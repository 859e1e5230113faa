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

`P2PExchange` / `P2PExpertParallelMoE` are the B200-native variant: the same
semantics over peer memory (csrc/ep_p2p.cu) -- the home rank's kernels store
pair rows straight into the owners' mailboxes (CUDA IPC-mapped, NVLink P2P on
an NVSwitch node) and the owners store outputs straight back, with
release/acquire flags at system scope instead of collectives: no host sync and
no counts all-to-all per layer.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .runtime import StepEngine


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


# ----------------------------------------------------------------------------- peer-memory exchange
class _DevView:
    """A torch view of raw device memory (the IPC-mapped mailbox)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class P2PExchange:
    """Dispatch / combine over peer memory (ep_p2p.cu; include/mobile.h).

    cap = rows one source may send one owner per exchange (T_max * k_max is
    the worst case).  Collective setup (mailbox handles all-gathered once);
    each exchange is kernels only, stream-ordered on the current stream."""

    def __init__(self, E: int, d: int, cap: int, group=None, device=None, bf16_rows: bool = False):
        """bf16_rows: dispatch the rows as bf16 (half the link bytes) -- for
        owners whose experts run on the tcgen05 path (bf16 activations)."""
        import ctypes as C

        from . import _native as N
        self.N = N
        self.group = group
        self.G = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.E, self.d, self.cap = E, d, cap
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        box = C.c_void_p()
        N.check(N.lib.mobile_ep_mailbox_create(self.G, cap, d, C.byref(box)), "ep mailbox")
        self.box = box.value
        handle = (C.c_ubyte * 64)()
        N.check(N.lib.mobile_ep_ipc_handle(C.c_void_p(self.box), handle), "ep ipc handle")
        handles = [bytes(handle)]
        if self.G > 1:
            handles = [None] * self.G
            dist.all_gather_object(handles, bytes(handle), group=group)
        self.opened = []
        ptrs = []
        for g in range(self.G):
            if g == self.rank:
                ptrs.append(self.box)
                continue
            p = C.c_void_p()
            hb = (C.c_ubyte * 64).from_buffer_copy(handles[g])
            N.check(N.lib.mobile_ep_ipc_open(hb, C.byref(p)), "ep ipc open")
            ptrs.append(p.value)
            self.opened.append(p.value)
        self.peers = torch.tensor(ptrs, dtype=torch.int64, device=dev)
        own, loc = owner_table(E, self.G, dev)
        self.owner, self.local_id = own.int().contiguous(), loc.int().contiguous()
        self.counts = torch.zeros(self.G, dtype=torch.int32, device=dev)
        self.flags = torch.zeros(1, dtype=torch.int32, device=dev)
        self.k_in = torch.zeros(self.G * cap, dtype=torch.int32, device=dev)
        self.epoch_dev = torch.zeros(1, dtype=torch.int32, device=dev)  # advanced on the device per exchange
        self._bufs: dict = {}
        # views of this rank's mailbox (layout of ep_p2p.cu Box)
        rows_b = (self.G * cap * d * 4 + 255) // 256 * 256
        ids_b = (self.G * cap * 4 + 255) // 256 * 256
        self.bf16_rows = bool(bf16_rows)
        if self.bf16_rows:  # bf16 rows packed at d * 2 bytes in the row area (no bf16 typestr: int16 view)
            self.in_rows = torch.as_tensor(_DevView(self.box, (self.G * cap, d), "<i2"), device=dev).view(torch.bfloat16)
        else:
            self.in_rows = torch.as_tensor(_DevView(self.box, (self.G * cap, d), "<f4"), device=dev)
        self.in_ids = torch.as_tensor(_DevView(self.box + rows_b, (self.G * cap,), "<i4"), device=dev)
        del ids_b

    def _s(self):
        return torch.cuda.current_stream().cuda_stream

    def exchange(self, h2: torch.Tensor, idx: torch.Tensor, k_tok: torch.Tensor, expert_fn,
                 timer: "ExchangeTimer | None" = None) -> torch.Tensor:
        """h2 (T, d) rows of this rank's tokens, idx (T, k_max) selections ->
        Y (T*k_max, d) expert outputs in pair order; expert_fn(rows, ids,
        k_tok) runs this rank's experts on its mailbox rows.  Kernels only,
        stream-ordered, no host sync; the epoch lives in device memory
        (advanced by the first kernel), so the exchange can be captured in a
        CUDA graph and replayed.  `timer` (eager only) records CUDA events
        around the dispatch / owner experts / return legs."""
        N, P_ = self.N, self.N.ptr
        T, k_max = idx.shape
        if T * k_max > self.cap:
            raise ValueError(f"P2PExchange: {T * k_max} pairs exceed the mailbox capacity {self.cap}")
        key = (T, k_max)
        if key not in self._bufs:
            self._bufs[key] = (torch.empty(T * k_max, dtype=torch.int32, device=self.dev),
                               torch.empty(T * k_max, self.d, dtype=torch.float32, device=self.dev))
        dest, Y = self._bufs[key]
        s = self._s()
        if timer is not None:
            timer.mark("start")
        N.check(N.lib.mobile_ep_advance(P_(self.epoch_dev), s), "ep advance")
        N.check(N.lib.mobile_ep_dispatch(P_(h2), P_(idx), P_(k_tok), T, k_max, self.d, P_(self.owner),
                                         P_(self.local_id), P_(self.peers), self.G, self.rank, self.cap, 0,
                                         P_(self.epoch_dev), int(self.bf16_rows), P_(dest), P_(self.counts),
                                         P_(self.flags), s),
                "ep dispatch")
        N.check(N.lib.mobile_ep_wait(self.box, self.G, self.cap, self.d, 0, 0, P_(self.epoch_dev), P_(self.k_in),
                                     P_(self.flags), s), "ep wait (in)")
        if timer is not None:
            timer.mark("dispatched")
        out = expert_fn(self.in_rows, self.in_ids, self.k_in)
        if timer is not None:
            timer.mark("experts")
        N.check(N.lib.mobile_ep_return(P_(out), self.box, P_(self.peers), self.G, self.rank, self.cap, self.d, 0,
                                       P_(self.epoch_dev), s), "ep return")
        N.check(N.lib.mobile_ep_wait(self.box, self.G, self.cap, self.d, 1, 0, P_(self.epoch_dev), None,
                                     P_(self.flags), s), "ep wait (back)")
        N.check(N.lib.mobile_ep_collect(self.box, P_(dest), T * k_max, self.G, self.cap, self.d, P_(Y), s),
                "ep collect")
        if timer is not None:
            timer.mark("returned")
        return Y

    def close(self):
        if getattr(self, "box", None) is None:
            return
        torch.cuda.synchronize()
        for p in self.opened:
            self.N.lib.mobile_ep_ipc_close(p)
        self.opened = []
        if self.G > 1:
            dist.barrier(group=self.group)  # every peer unmapped this mailbox
        self.N.lib.mobile_ep_mailbox_destroy(self.box)
        self.box = None


class ExchangeTimer:
    """CUDA events around the legs of eager exchanges (dispatch + wait,
    owner experts, return + wait + collect), summed per leg."""

    LEGS = (("start", "dispatched", "dispatch"), ("dispatched", "experts", "owner_experts"),
            ("experts", "returned", "return"))

    def __init__(self):
        self.events: list[dict] = []
        self.cur: dict | None = None

    def mark(self, name: str):
        if name == "start":
            self.cur = {}
            self.events.append(self.cur)
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.cur[name] = e

    def summary_ms(self) -> dict:
        torch.cuda.synchronize()
        out = {leg: 0.0 for _, _, leg in self.LEGS}
        for ev in self.events:
            for a, b, leg in self.LEGS:
                out[leg] += ev[a].elapsed_time(ev[b])
        out["exchanges"] = len(self.events)
        return out


class P2PExpertParallelMoE(ExpertParallelMoE):
    """ExpertParallelMoE with the peer-memory exchange (same decisions, gates
    and combine on the home rank; the owner runs its experts on its mailbox)."""

    def __init__(self, moe_full_router, local_moe, E: int, d: int, cap: int, group=None):
        self.router_moe = moe_full_router
        self.local = local_moe
        self.x = P2PExchange(E, d, cap, group, bf16_rows=local_moe.tc_ok)

    def forward(self, x, layer, k_tok, k_max, replay=None, replay_mask=None, reuse_gates=False, ln_out=None):
        return self.forward_sc(x, layer, k_tok, k_max, replay=replay, replay_mask=replay_mask,
                               reuse_gates=reuse_gates, ln_out=ln_out)[0]

    def forward_sc(self, x, layer, k_tok, k_max, replay=None, replay_mask=None, reuse_gates=False, ln_out=None):
        """forward() plus the router scratch (logits, selections): the
        DecodeSession layer interface (MoBiLEMoE.forward)."""
        from . import kernels as K
        rm = self.router_moe
        sc = rm.route(x, layer, k_tok, k_max, replay=replay, replay_mask=replay_mask, reuse_gates=reuse_gates)
        r = sc["router"]

        def experts(rows, ids, k_in):  # one kernel choice for any row count: G-invariant outputs
            return self.local.rows_ffn(layer, rows, ids, k_in, clone=False, force_tc=self.local.tc_ok)

        Y = self.x.exchange(r["h2"], r["idx"], k_tok, experts)
        Ys = rm.shared_rows(layer, r["h2"], sc) if rm.S else None
        shared_logits = r["extra"] if rm.dw.n_gate_rows else None
        return K.combine(x, Y, r["gates"], k_tok, Ys, rm.S, shared_logits, ln_out=ln_out), sc



class EPStepEngine(StepEngine):
    """Expert-parallel decode engine: a StepEngine whose
    routed experts are sharded over the ranks of `group` and exchanged over
    peer memory every layer.

    Each rank decodes its own B sequences (data-parallel over the batch):
    embed, attention, router, top-k / replay, shared experts, combine and the
    head run on the home rank with the single-GPU kernels; only the routed
    expert rows travel (P2PExchange: dispatch into the owners' mailboxes, the
    owner's experts on the tcgen05 grouped GEMM for any row count, outputs
    back, combine in selection order).  Every output row is a function of its
    own input row alone, so a rank's tokens, router logits, selections and
    confidences are bit-identical for any G (tests/test_ep_engine_gpu.py).
    The exchange is kernels only with a device-side epoch, so each pass kind
    is captured in one CUDA graph like the single-GPU engine.

    `dm` holds the replicated weights (its routed experts are not read);
    `local` is a MoBiLEMoE over this rank's expert block
    (DeviceWeights.shard_experts)."""

    def __init__(self, dm, local, batch: int, max_len: int, group=None, graphs: bool = True, gemm=None,
                 shard_runtime=None):
        """shard_runtime: an OffloadRuntime over this rank's expert shard (its
        routed experts in pinned host memory behind the rank's own HBM expert
        cache, so the cache capacity of the job is G x the per-rank budget).
        The owner then reads back, per layer, which of its experts it
        received (one small D2H + host sync, the on-demand protocol of
        engine.py:243-244 on the owner), requests + pins them in its cache,
        copies the misses and runs its rows from the cache slots; eager
        passes only (the host sits between the exchange's legs)."""
        if shard_runtime is not None:
            graphs = False
        super().__init__(dm, batch, max_len, graphs=graphs, persistent=False, gemm=gemm)
        self.fork_shared = False  # _experts below runs the shared experts itself
        s = dm.spec
        self.ep_local = local
        self.ep_rt = shard_runtime
        if shard_runtime is not None:
            cap = batch * s.k_big
            G = dist.get_world_size(group) if dist.is_initialized() else 1
            self._ids_h = torch.zeros(G * cap, dtype=torch.int32, pin_memory=True)
            self._kin_h = torch.zeros(G * cap, dtype=torch.int32, pin_memory=True)
        self.ep_group = group
        self._pf = None  # prompt-sized exchange (prefill), created on first use
        self.xch = P2PExchange(s.num_experts, s.hidden_dim, batch * s.k_big, group, dm.device, bf16_rows=local.tc_ok)
        self.ex_timer: ExchangeTimer | None = None  # eager mode: CUDA events around the exchange legs

    def _experts(self, l: int, kind: str, sc: dict, loc, shared_join=None) -> torch.Tensor:
        from . import kernels as K
        rm, local = self.dm.moe, self.ep_local
        r = sc["router"]
        k_tok = self.k_tok[kind]

        def experts(rows, ids, k_in):
            if self.ep_rt is None:
                return local.rows_ffn(l, rows, ids, k_in, clone=False, force_tc=local.tc_ok)
            # owner with an offloaded shard: the received experts (sorted, distinct) -> its cache
            self._ids_h.copy_(ids, non_blocking=True)
            self._kin_h.copy_(k_in, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            self.ep_rt.sync_point()
            got = sorted({int(e) for e, v in zip(self._ids_h.tolist(), self._kin_h.tolist()) if v})
            # a rank that received no rows this layer still needs the cache's
            # slot table (no expert is active, nothing is read through it);
            # the resident location does not exist for an offloaded shard
            loc = self.ep_rt._require(l, got, 0) if got else self.ep_rt._location(l, 0)
            out = local.rows_ffn(l, rows, ids, k_in, clone=False, force_tc=local.tc_ok, loc=loc)
            if got:
                self.ep_rt._release(l, got)
            return out

        Y = self.xch.exchange(r["h2"], r["idx"], k_tok, experts, timer=None if self.use_graphs else self.ex_timer)
        Ys = rm.shared_rows(l, r["h2"], sc) if rm.S else None
        shared_logits = r["extra"] if rm.dw.n_gate_rows else None
        return K.combine(self.xa, Y, r["gates"], k_tok, Ys, rm.S, shared_logits, x_out=sc["x_out"], ln_out=self.ln)

    def prefill(self, prompt: list[int], prefill_k: int | None = None):
        """The prompt through the session path with the MoE layers expert-
        parallel (collective: every rank prefills, in lockstep); the exchange
        for prompt-sized batches is created on first use (capacity = the
        prompt's pairs)."""
        s = self.spec
        n = max(len(prompt) - 1, 1)
        kpf = s.k_big if prefill_k is None else prefill_k
        if self._pf is None or self._pf.x.cap < n * kpf:
            if self._pf is not None:
                self._pf.x.close()
            self._pf = P2PExpertParallelMoE(self.dm.moe, self.ep_local, s.num_experts, s.hidden_dim, cap=n * kpf,
                                            group=self.ep_group)
        self.sess.moe_forward = self._pf.forward_sc
        try:
            super().prefill(prompt, prefill_k)
        finally:
            self.sess.moe_forward = None

    def run_pass(self, kind: str):
        super().run_pass(kind)
        if self.ep_rt is not None:  # every request of the pass is settled before the next one
            self.stream.synchronize()
            self.ep_rt.token_end()

    def close(self):
        self.xch.close()
        if self._pf is not None:
            self._pf.x.close()
            self._pf = None
