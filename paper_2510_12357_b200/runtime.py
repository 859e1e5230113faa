"""Graph-captured decode step (the B200 hot loop around the MoBiLE layer).

One decode step of B sequences is built from libmobile kernels only -- embed,
per layer [LN+QKV GEMV, KV-cache attention, O GEMV + residual, fused router /
top-k / replay, permute, grouped expert GEMVs, shared experts, combine], head +
confidence -- with every position read from device memory, so each pass kind
is captured once in CUDA graphs and replayed per token:

  little : k_little experts, own routing                  (toymoe.little_forward)
  big    : k_big experts, selection replayed from the little
           pass's recorded logits (h_s)                      (toymoe.big_forward)
  full   : k_big experts, own routing (full-top-k baseline)   (toymoe.full_forward)

HBM-resident experts: a pass is ONE graph launch.  Offloaded experts: a pass
is L+1 graph segments cut at each layer's routing, because the on-demand
passes need the layer's selection on the host to issue expert copies
(engine.py:243-244); the segment boundary is the single host sync per layer.
Each segment starts with the H2D of the layer's slot table (a memcpy node
reading pinned host memory written by the C++ cache runtime) and ends with
the D2H of the next layer's active-expert list.  The replayed big pass needs
no sync at all: its plan is known up front (policy.py:86-106), so all its
segments, prefetches and waits are enqueued back to back.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import _native as N
from . import kernels as K
from .model import FFN_IMPL, TC_MIN_TOKENS, DecodeSession, DeviceModel, pos_rows
from .policy import plan_from_targets

KINDS = ("little", "big", "full")
GEMV_MAX_BATCH = 4  # largest batch on the GEMV decode path (stream GEMV / persistent pass tile)
GEMM_MIN_BATCH = 5  # resident bf16 decode switches to the GEMM path from here (scripts/batch_paths.py, round 2)
MAX_BATCH = 1024
PREFILL_GRAPHS_MAX = 4  # captured prefill graphs kept per engine (one per prompt length, oldest dropped)


class StepEngine:
    def __init__(self, dm: DeviceModel, batch: int, max_len: int, runtime=None, graphs: bool = True,
                 persistent: bool | None = None, zero_sync: bool | None = None, gemm: bool | None = None):
        s = dm.spec
        # small batches: the GEMV decode path (persistent pass / bulk-copy
        # streaming); larger ones run projections, experts and head as tcgen05
        # GEMMs (default from GEMM_MIN_BATCH when the shapes allow it)
        if gemm is None:
            gemm = batch > GEMV_MAX_BATCH or (batch >= GEMM_MIN_BATCH and runtime is None and dm.moe.tc_ok
                                              and persistent is not True)
        self.gemm_path = bool(gemm)
        # batched GEMM path: each layer's shared experts run on a side stream
        # concurrently with routing and the routed experts (C4 B = 8 / 64 / 256)
        # (only when the batch's experts run on the grouped GEMM: a GEMM path
        # forced below TC_MIN_TOKENS streams its shared experts with the routed
        # ones, and a fork there was never joined -- graph capture failed)
        self.fork_shared = (self.gemm_path and dm.moe.S > 0 and dm.moe.tc_ok and batch >= TC_MIN_TOKENS
                            and FFN_IMPL != "stream_only" and os.environ.get("MOBILE_SHARED_FORK", "1") != "0")
        self.side = torch.cuda.Stream(device=dm.device) if self.fork_shared else None
        # opt-in (MOBILE_ROUTER_PF=1): the router launch starts the selected
        # experts' whole gate-up weights toward L2.  Measured 2-8x SLOWER
        # (per-op little pass C2 1.02 -> 3.14 ms, C3 1.86 -> 4.08, C5 4.02 ->
        # 33.96; profiles/r2_ab_routerpf.txt): the prefetch doubles the
        # experts' HBM traffic and thrashes L2 for experts larger than it
        self.router_prefetch = (runtime is None and not self.gemm_path
                                and os.environ.get("MOBILE_ROUTER_PF", "0") == "1")
        # resident batches 1-4: the per-op engine (graph-replayed, PDL-chained
        # kernels; split-KV attention; 16-warp streaming GEMV) beats or ties the
        # persistent pass (scripts/batch_paths.py, round 2, little / full pass:
        # B = 1 C2 1.01 / 1.20 vs 1.17 / 1.46 ms, C4 1.84 / 2.14 vs 2.06 / 2.46;
        # B = 2 C2 1.47 / 1.99 vs 1.60 / 2.14, C4 2.74 / 3.67 vs 2.79 / 3.57;
        # B = 3-4 also ahead of the GEMM path; profiles/r2_batch_paths_gemv16.txt).
        # The persistent pass stays the engine of offloaded experts (zero-sync)
        if persistent is None and runtime is None and not self.gemm_path:
            persistent = False
        if self.gemm_path:
            if not dm.moe.tc_ok:
                raise ValueError(f"StepEngine: batch {batch} > {GEMV_MAX_BATCH} needs the tcgen05 GEMM path "
                                 f"(bf16 SwiGLU shapes)")
            if runtime is not None:
                raise ValueError(f"StepEngine: offloaded experts need batch <= {GEMV_MAX_BATCH}")
            if batch > MAX_BATCH:
                raise ValueError(f"StepEngine: batch {batch} > {MAX_BATCH}")
        self.dm, self.spec, self.B, self.max_len = dm, s, batch, max_len
        self.rt = runtime
        self.use_graphs = graphs
        dev = dm.device
        L, E, d, B = s.num_layers, s.num_experts, s.hidden_dim, batch
        self.sess = DecodeSession(dm, batch, max_len)
        f32, i32 = torch.float32, torch.int32
        self.pe = pos_rows(s, max_len, 0, dev).contiguous()
        self.tok = torch.zeros(B, dtype=i32, device=dev)
        self.pos = torch.zeros(B, dtype=i32, device=dev)
        self.tok_host = torch.zeros(B, dtype=i32, pin_memory=True)
        self.x = torch.empty(B, d, dtype=f32, device=dev)
        self.ln = torch.empty(B, d, dtype=f32, device=dev)  # LN of the layer input (from embed / combine)
        self.qkv_rows = d + 2 * s.kv_dim  # [q | k | v] (k, v narrower under grouped-query attention)
        self.qkv = torch.empty(B, self.qkv_rows, dtype=f32, device=dev)
        self.att = torch.empty(B, d, dtype=f32, device=dev)
        self.xa = torch.empty(B, d, dtype=f32, device=dev)
        # this engine's own split-KV workspace (its stream and graphs only)
        self.attn_ws = K.attn_split_workspace(B, d, s.n_heads, max_len, dev)
        self.k = {"little": s.k_little, "big": s.k_big, "full": s.k_big}
        self.k_tok = {kd: torch.full((B,), self.k[kd], dtype=i32, device=dev) for kd in KINDS}
        # zero-initialised: the graph warm-up replays states["little"] before any real pass
        self.states = {kd: torch.zeros(L, B, E, dtype=f32, device=dev) for kd in KINDS}
        self.idx = {kd: torch.empty(L, B, self.k[kd], dtype=i32, device=dev) for kd in KINDS}
        self.ones = torch.ones(B, dtype=torch.uint8, device=dev)
        self.head = {kd: dict(conf=torch.empty(B, dtype=f32, device=dev), argmax=torch.empty(B, dtype=i32, device=dev),
                              fallback=torch.empty(B, dtype=torch.uint8, device=dev)) for kd in KINDS}
        self.head_ws = K.StreamHeadWorkspace(dev)
        if self.gemm_path:
            self.xb = torch.empty(B, d, dtype=torch.bfloat16, device=dev)  # bf16 GEMM operand
            self.logits = torch.empty(B, s.vocab_size, dtype=f32, device=dev)
        self.gamma = torch.zeros(1)  # host value baked at capture; see set_gamma
        self._gamma = 0.7
        self.graphs: dict = {}
        self.stream = torch.cuda.Stream(device=dev)
        if runtime is not None:
            self.active_host = torch.zeros(L, E + 1, dtype=i32, pin_memory=True)
        self.reuse_gates = False
        self.prefill_graphs = True  # capture one prefill graph per prompt length (resident experts)
        self._pf_graphs: dict = {}
        self.timer = None  # kernel timer (eager mode only: events are not graph nodes here)
        # persistent decode-pass kernel (decode_pass.cu): one launch per pass /
        # offload segment.  None = use it whenever the shape is supported.
        self.persistent = persistent
        self.dp = {}
        self.record_passes = False  # metrics.measure_stream
        self.pass_log: list = []
        # zero-sync offload (persistent + offloaded experts): one launch per pass,
        # the C++ cache driver answers each layer's published selection while
        # the kernel runs (decode_pass.cu mobile_dp_run_offload_pass)
        self.zero_sync = zero_sync if zero_sync is not None else os.environ.get("MOBILE_ZS", "1") != "0"

    # ------------------------------------------------------------------ kernels
    def _attn(self, l: int, x_in: torch.Tensor) -> torch.Tensor:
        """q,k,v = LN(x) Wqkv (self.ln holds LN(x_in)); attention; x + att Wo."""
        dw, s = self.dm.dw, self.spec
        d, B = s.hidden_dim, self.B
        if self.gemm_path:
            return self._attn_gemm(l, x_in)
        wc = self.dm.moe.wcode
        K.stream_gemv([K.sg_group(w_base=dw.qkv[l].data_ptr(), K=d, rows=self.qkv_rows, x=self.ln, dense_T=B,
                                  out=self.qkv)], wc, B)
        K.attn_decode(self.qkv, self.sess.kc[l], self.sess.vc[l], self.pos, s.n_heads, out=self.att, ws=self.attn_ws)
        K.stream_gemv([K.sg_group(w_base=dw.o[l].data_ptr(), K=d, rows=d, x=self.att, dense_T=B, out=self.xa,
                                  residual=x_in)], wc, B)
        return self.xa

    def _dense_gemm(self, w: torch.Tensor, n_out: int, out: torch.Tensor, epi: int):
        """out (B, n_out) [+]= xb @ w^T on the tcgen05 grouped GEMM (dense mode)."""
        d, B = self.spec.hidden_dim, self.B
        tiles = (B + 127) // 128 * (n_out // 128)
        K.grouped_gemm(self.xb, d, w.data_ptr(), w.numel() * w.element_size(), 1, n_out, max_tiles=tiles,
                       dense_rows=B, dense_experts=1, epi=epi, out_f32=out, ldo=n_out)

    def _attn_gemm(self, l: int, x_in: torch.Tensor) -> torch.Tensor:
        """Large batch: QKV and O projections as tcgen05 GEMMs (bf16 operands,
        f32 accumulate), the O projection accumulated onto the residual."""
        dw, d, B = self.dm.dw, self.spec.hidden_dim, self.B
        K.gather_bf16(self.ln, None, 1, B, self.xb)
        self._dense_gemm(dw.qkv[l], self.qkv_rows, self.qkv, K.GG_STORE_F32)
        K.attn_decode(self.qkv, self.sess.kc[l], self.sess.vc[l], self.pos, self.spec.n_heads, out=self.att,
                      ws=self.attn_ws)
        K.gather_bf16(self.att, None, 1, B, self.xb)
        self.xa.copy_(x_in)
        self._dense_gemm(dw.o[l], d, self.xa, K.GG_ACCUM_F32)
        return self.xa

    def _route(self, l: int, kind: str) -> dict:
        moe = self.dm.moe
        replay = self.states["little"][l] if kind == "big" else None
        mask = self.ones if kind == "big" else None
        return moe.route(self.xa, l, self.k_tok[kind], self.k[kind], replay=replay, replay_mask=mask,
                         reuse_gates=self.reuse_gates and kind == "big",
                         logits_out=self.states[kind][l], idx_out=self.idx[kind][l],
                         prefetch_experts=self.router_prefetch)

    def _experts(self, l: int, kind: str, sc: dict, loc, shared_join=None) -> torch.Tensor:
        return self.dm.moe.experts(self.xa, l, sc, self.k_tok[kind], self.k[kind], loc,
                                   timer=None if self.use_graphs else self.timer, ln_out=self.ln,
                                   shared_join=shared_join)

    def _head(self, x_last: torch.Tensor, kind: str):
        """LN(x) is already in self.ln (written by the last layer's combine)."""
        s = self.spec
        if self.gemm_path:
            K.gather_bf16(self.ln, None, 1, self.B, self.xb)
            self._dense_gemm(self.dm.dw.head, s.vocab_size, self.logits, K.GG_STORE_F32)
            K.logits_confidence(self.logits, s.logit_scale, self._gamma, self.head[kind])
            return
        K.stream_head(self.ln, self.dm.dw.head, self._gamma, s.logit_scale, ws=self.head_ws, out=self.head[kind])

    def _offload_loc(self, l: int, kind: str):  # noqa: D401
        row = 1 if kind == "big" else 0
        return self.rt._location(l, row), row

    # ------------------------------------------------------------------ segments
    def _seg(self, kind: str, l: int):
        """Segment l of an offloaded pass: experts(l-1) [+ attn/route(l)]."""
        L = self.spec.num_layers
        if self.dp:
            row = 1 if kind == "big" else 0
            if l > 0:
                K.memcpy_async(self.rt.slot_dev[row, l - 1], self.rt.slot_host[row, l - 1])
            self._dp_launch(kind, l)
            if l < L and kind != "big":
                K.memcpy_async(self.active_host[l], self.active_dev[l])
            return
        if l == 0:
            K.embed(self.tok, self.pos, self.dm.dw.embed, self.pe, self.x, ln_out=self.ln)
            x_in = self.x
        else:
            loc, row = self._offload_loc(l - 1, kind)
            K.memcpy_async(self.rt.slot_dev[row, l - 1], self.rt.slot_host[row, l - 1])
            x_in = self._experts(l - 1, kind, self._sc[kind][l - 1], loc)
        if l == L:
            self._head(x_in, kind)
            return
        self._attn(l, x_in)
        sc = self._route(l, kind)
        self._sc[kind][l] = sc
        if kind != "big":
            K.memcpy_async(self.active_host[l], sc["perm"]["active"])

    # ------------------------------------------------------------------ persistent pass
    def _dp_build(self, gamma: float, reuse_gates: bool) -> bool:
        """Create one mobile_dp program per pass kind; False if unsupported."""
        s, dw, B, dev = self.spec, self.dm.dw, self.B, self.dm.device
        L, E, d = s.num_layers, s.num_experts, s.hidden_dim
        f32, i32 = torch.float32, torch.int32
        ng = dw.n_gate_rows
        kb = s.k_big
        self.q = torch.empty(B, d, dtype=f32, device=dev)
        self.extra = torch.zeros(L, B, max(ng, 1), dtype=f32, device=dev)
        self.gates = {kd: torch.empty(L, B, self.k[kd], dtype=f32, device=dev) for kd in KINDS}
        self.dpU = torch.empty(B * kb, s.ffn, dtype=f32, device=dev)
        self.dpY = torch.empty(B * kb, d, dtype=f32, device=dev)
        S = s.n_shared
        self.dpUs = torch.empty(max(B * S, 1), max(s.shared_ffn, 1), dtype=f32, device=dev)
        self.dpYs = torch.empty(max(B * S, 1), d, dtype=f32, device=dev)
        self.active_dev = torch.zeros(L, E + 1, dtype=i32, device=dev)
        self.dp_flags = torch.zeros(1, dtype=i32, device=dev)
        self._dp_models = {}
        for kd in KINDS:
            m = N.mobile_dp_model()
            m.B, m.L, m.d, m.H, m.V, m.E, m.k = B, L, d, s.n_heads, s.vocab_size, E, self.k[kd]
            m.Hkv = s.kv_heads
            m.n_shared, m.n_gate, m.ffn, m.shared_ffn = S, ng, s.ffn, s.shared_ffn if S else 0
            m.activation = self.dm.moe.act
            m.gate_norm = self.dm.moe.gate_norm
            m.reuse_gates = int(bool(reuse_gates))
            m.w_dtype = self.dm.moe.wcode
            m.max_len = self.max_len
            m.offload = int(self.rt is not None)
            m.logit_scale, m.gamma = float(s.logit_scale), float(gamma)
            m.qkv, m.o, m.router, m.head = dw.qkv.data_ptr(), dw.o.data_ptr(), dw.router.data_ptr(), dw.head.data_ptr()
            if S:
                m.shared = dw.shared.data_ptr()
                m.shared_stride = dw.shared_bytes
                m.shared_w2_offset = dw.s_w13_elems * dw.elem_bytes
            if self.rt is None:
                m.experts = dw.experts.data_ptr()
                m.expert_layer_stride = E * dw.expert_bytes
                m.slot_table = None
            else:
                m.experts = self.rt.pool.data_ptr()
                m.expert_layer_stride = 0
                m.slot_table = self.rt.slot_dev[1 if kd == "big" else 0].data_ptr()
            m.expert_stride = dw.expert_bytes
            m.expert_w2_offset = dw.w13_elems * dw.elem_bytes
            m.embed, m.pe = dw.embed.data_ptr(), self.pe.data_ptr()
            m.tok, m.pos = self.tok.data_ptr(), self.pos.data_ptr()
            m.kc, m.vc = self.sess.kc.data_ptr(), self.sess.vc.data_ptr()
            m.x, m.xa, m.q, m.att = self.x.data_ptr(), self.xa.data_ptr(), self.q.data_ptr(), self.att.data_ptr()
            m.U, m.Us, m.Y, m.Ys = self.dpU.data_ptr(), self.dpUs.data_ptr(), self.dpY.data_ptr(), self.dpYs.data_ptr()
            m.states, m.extra = self.states[kd].data_ptr(), self.extra.data_ptr()
            m.replay = self.states["little"].data_ptr() if kd == "big" else None
            m.idx_out, m.gates_out = self.idx[kd].data_ptr(), self.gates[kd].data_ptr()
            m.active_out = self.active_dev.data_ptr()
            m.head_logits = None
            h = self.head[kd]
            m.conf, m.argmax, m.fallback = h["conf"].data_ptr(), h["argmax"].data_ptr(), h["fallback"].data_ptr()
            m.flags = self.dp_flags.data_ptr()
            handle = C.c_void_p()
            st = N.lib.mobile_dp_create(C.byref(m), C.byref(handle))
            if st != N.OK:
                for hh in self.dp.values():
                    N.lib.mobile_dp_destroy(hh)
                self.dp = {}
                if self.persistent:  # explicitly requested
                    N.check(st, "decode_pass create")
                return False
            self.dp[kd] = handle
            self._dp_models[kd] = m
        return True

    def dp_info(self, kind: str = "little") -> dict:
        out = (C.c_int * 4)()
        N.lib.mobile_dp_info(self.dp[kind], out)
        return dict(phases=out[0], stages=out[1], smem=out[2], grid=out[3])

    def _dp_launch(self, kind: str, segment: int):
        K._count()
        N.check(N.lib.mobile_dp_launch(self.dp[kind], segment, torch.cuda.current_stream().cuda_stream),
                "decode_pass launch")

    def __del__(self):
        if getattr(N, "lib", None) is not None:
            for h in getattr(self, "dp", {}).values():
                N.defer_destroy("mobile_dp_destroy", h)
        self.dp = {}

    def _whole_pass(self, kind: str):
        """A pass with HBM-resident experts (one graph)."""
        if self.dp:
            self._dp_launch(kind, -1)
            return
        K.embed(self.tok, self.pos, self.dm.dw.embed, self.pe, self.x, ln_out=self.ln)
        x_in = self.x
        for l in range(self.spec.num_layers):
            self._attn(l, x_in)
            join = self._shared_fork(l, kind) if self.fork_shared else None
            sc = self._route(l, kind)
            x_in = self._experts(l, kind, sc, None, shared_join=join)
        self._head(x_in, kind)

    def _shared_fork(self, l: int, kind: str):
        """Batched (GEMM-path) pass: the layer's shared experts start from the
        post-attention residual on a side stream while the main stream routes
        and runs the routed experts; the returned join makes the main stream
        wait for them before the combine (captured as fork / join edges)."""
        main = torch.cuda.current_stream()
        self.side.wait_stream(main)
        with torch.cuda.stream(self.side):
            self.dm.moe.shared_from_residual(self.xa, l, self.B, self.k[kind])
        return lambda: main.wait_stream(self.side)

    def _capture(self, key, fn):
        if not self.use_graphs:
            return fn
        g = torch.cuda.CUDAGraph()
        # warm up once eagerly (sets kernel attributes, allocates scratch)
        with torch.cuda.stream(self.stream):
            fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=self.stream):
            fn()
        self.graphs[key] = g
        return g.replay

    def build(self, gamma: float = 0.7, reuse_gates: bool = False):
        """Capture the graphs for every pass kind (gamma / reuse are baked in)."""
        self._gamma, self.reuse_gates = gamma, reuse_gates
        N.reap()  # destroys queued by finalizers: never inside the captures below
        # buffers were zero-filled on the caller's stream; the warm-up runs on ours
        self.stream.wait_stream(torch.cuda.current_stream())
        L = self.spec.num_layers
        for h in self.dp.values():
            N.lib.mobile_dp_destroy(h)
        self.dp = {}
        if self.persistent is not False and self.timer is None and not self.gemm_path:
            self._dp_build(gamma, reuse_gates)
        self._sc = {kd: [None] * L for kd in KINDS}
        self.run = {}
        if self.rt is None:
            for kd in KINDS:
                self.run[kd] = self._capture(kd, lambda kd=kd: self._whole_pass(kd))
        else:
            # offload: warm-up needs valid slot tables; point every table at slot 0
            self.rt.slot_dev.zero_()
            self.rt.slot_host.zero_()
            for kd in KINDS:
                self.run[kd] = [self._capture((kd, l), lambda kd=kd, l=l: self._seg(kd, l)) for l in range(L + 1)]
        torch.cuda.synchronize()
        if self.dp:
            self.dp_flags.zero_()
        return self

    # ------------------------------------------------------------------ passes
    def _launch(self, fn):
        with torch.cuda.stream(self.stream):
            fn()

    def pass_resident(self, kind: str):
        self._launch(self.run[kind])

    def _pass_offload_zs(self, kind: str):
        """Whole offloaded pass in one persistent launch; the C++ driver runs
        the cache protocol against the running kernel (no per-layer sync)."""
        rt, s = self.rt, self.spec
        planned = kind == "big"
        targets, k = None, 0
        if planned:
            with torch.cuda.stream(self.stream):
                idx, _ = K.topk_rows(self.states["little"][:, 0].contiguous(), s.k_big)
                flat = idx.cpu().reshape(-1).tolist()  # one D2H for the whole planned pass
            k = s.k_big
            targets = (C.c_int * len(flat))(*flat)
        fresh = C.c_int()
        K._count()
        N.check(N.lib.mobile_dp_run_offload_pass(self.dp[kind], rt.h, int(planned), targets, k, rt.lookahead,
                                                 self.stream.cuda_stream, C.byref(fresh)), "zero-sync offload pass")
        rt.fresh += fresh.value

    def pass_offload(self, kind: str):
        """Drive the L+1 segments with the engine.py:121-169 protocol: in C++
        (mobile_offload_run_pass) when the segments are captured graphs, else
        from Python (eager mode, used for per-kernel instrumentation).  With the
        persistent kernel and zero_sync: one launch per pass."""
        if self.dp and self.zero_sync:
            return self._pass_offload_zs(kind)
        if self.use_graphs:
            return self._pass_offload_native(kind)
        rt, L = self.rt, self.spec.num_layers
        segs = self.run[kind]
        row = 1 if kind == "big" else 0
        st = C.c_int()
        if kind == "big":
            with torch.cuda.stream(self.stream):
                idx, _ = K.topk_rows(self.states["little"][:, 0].contiguous(), self.spec.k_big)
                targets = idx.cpu().tolist()  # one D2H for the whole planned pass
            waiting = list(plan_from_targets(targets, rt.lookahead).entries)
        prev = None
        for l in range(L):
            self._launch(segs[l])  # experts(l-1), (2) attention(l), routing(l)
            if prev is not None:  # (6) unpin l-1 before layer l's window (engine.py:152-153, 131)
                self._release(l - 1, prev)
            if kind == "big":  # (1) issue window at the layer boundary (engine.py:98-119)
                kept = []
                for i, e in enumerate(waiting):
                    if e.earliest_issue_layer > l:
                        kept.extend(waiting[i:])
                        break
                    if e.expert.layer < l:
                        continue
                    rc = N.lib.mobile_offload_prefetch(rt.h, e.expert.layer, e.expert.expert, C.byref(st))
                    if rc == N.ERR_DEFERRED:
                        kept.append(e)
                    else:
                        N.check(rc, "offload prefetch")
                waiting = kept
            if kind == "big":
                experts = targets[l]
            else:  # on demand: the layer's selection comes back to the host
                self.stream.synchronize()
                N.lib.mobile_offload_sync(rt.h)
                a = self.active_host[l]
                experts = a[1:1 + int(a[0])].tolist()
            # (3) request + pin, issue misses, (4) compute stream waits on their copies
            self._require(l, experts, row)
            prev = experts
        self._launch(segs[L])  # (5) experts(L-1) + head
        self._release(L - 1, prev)

    def _pass_offload_native(self, kind: str):
        rt, s = self.rt, self.spec
        L = s.num_layers
        if not hasattr(self, "_execs"):
            self._execs = {kd: (C.c_ulonglong * (L + 1))(*[self.graphs[(kd, l)].raw_cuda_graph_exec()
                                                            for l in range(L + 1)]) for kd in KINDS}
        row = 1 if kind == "big" else 0
        planned = kind == "big"
        targets = None
        k = 0
        if planned:
            with torch.cuda.stream(self.stream):
                idx, _ = K.topk_rows(self.states["little"][:, 0].contiguous(), s.k_big)
                flat = idx.cpu().reshape(-1).tolist()  # one D2H for the whole planned pass
            k = s.k_big
            targets = (C.c_int * len(flat))(*flat)
        fresh = C.c_int()
        N.check(N.lib.mobile_offload_run_pass(
            rt.h, self._execs[kind], L, self.stream.cuda_stream, int(planned),
            None if planned else self.active_host.data_ptr(), targets, k, rt.slot_host[row].data_ptr(),
            None, 0, rt.lookahead, C.byref(fresh)), "offload run_pass")
        rt.fresh += fresh.value

    def _require(self, l, experts, row):
        rt = self.rt
        arr = (C.c_int * len(experts))(*experts)
        issued = C.c_int()
        N.check(N.lib.mobile_offload_require(rt.h, l, arr, len(experts), self.stream.cuda_stream,
                                             rt.slot_host[row, l].data_ptr(), C.byref(issued)), "offload require")
        rt.fresh += issued.value

    def _release(self, l, experts):  # (6) unpin + last-use events (engine.py:152-153)
        arr = (C.c_int * len(experts))(*experts)
        N.check(N.lib.mobile_offload_release(self.rt.h, l, arr, len(experts), self.stream.cuda_stream),
                "offload release")

    def run_pass(self, kind: str):
        # work the caller enqueued on its current stream (state fills) precedes the pass
        self.stream.wait_stream(torch.cuda.current_stream())
        rec = getattr(self, "record_passes", False)
        if rec:  # metrics.measure_stream: device time + cache accounting of this pass
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
            fresh0 = self.rt.fresh if self.rt else 0
            xfer0 = self.rt.counters()[1] if self.rt else 0
        if self.rt is None:
            self.pass_resident(kind)
        else:
            self.pass_offload(kind)
        if rec:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(self.stream)
            demand = self.spec.num_layers * self.k[kind] * self.B  # required requests of the pass
            misses = (self.rt.fresh - fresh0) if self.rt else 0
            fresh = (self.rt.counters()[1] - xfer0) if self.rt else 0
            self.pass_log.append((kind, e0, e1, demand - misses, misses, fresh))

    # ------------------------------------------------------------------ decode API
    def prefill(self, prompt: list[int], prefill_k: int | None = None):
        """Context positions [0, n-1) through the torch-free-of-graphs session
        path (T = n-1 tokens), then the last prompt token becomes the first
        step's input."""
        if self.B != 1:
            raise ValueError("prefill: batch-1 engine")
        s = self.spec
        kpf = s.k_big if prefill_k is None else prefill_k
        ctx = list(prompt[:-1])
        self.sess.pos = 0
        if ctx:
            n = len(ctx)
            # resident experts: the prompt's kernels are one CUDA graph per
            # prompt length (captured after the first eager prefill of that
            # length; the prompt ids are read from a static device buffer)
            key = (n, kpf)
            capturable = (self.use_graphs and self.rt is None and self.sess.moe_forward is None
                          and self.prefill_graphs)
            if capturable and key in self._pf_graphs:
                g, tbuf = self._pf_graphs[key]
                tbuf.copy_(torch.tensor([ctx], dtype=torch.long), non_blocking=False)
                self.stream.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(self.stream):
                    g.replay()
                self.sess.pos = n
            else:
                t = torch.tensor([ctx], dtype=torch.long, device=self.dm.device)
                k = torch.full((n,), kpf, dtype=torch.int32, device=self.dm.device)
                hook = self.rt.demand_hook("prefill") if self.rt else None
                with torch.cuda.stream(self.stream):
                    self.sess.run(t, k, kpf, expert_hook=hook)
                if self.rt:
                    self.stream.synchronize()
                    self.rt.token_end()
                if capturable:  # capture this length for the next prefills (the eager run warmed it up)
                    self.stream.synchronize()
                    tbuf = t.clone()
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=self.stream):
                        self.sess.pos = 0
                        self.sess.run(tbuf, k, kpf)
                    self._pf_graphs[key] = (g, tbuf)
                    while len(self._pf_graphs) > PREFILL_GRAPHS_MAX:  # bounded: drop the oldest length
                        self._pf_graphs.pop(next(iter(self._pf_graphs)))
                    self.sess.pos = n
        self.pos.fill_(len(ctx))
        self.tok.fill_(prompt[-1])
        torch.cuda.synchronize()

    def step(self, forced_fallback: bool | None = None, full: bool = False, next_token: int | None = None):
        """One decoded token (batch 1).  Returns (token, fell_back)."""
        rt = self.rt
        if full:
            self.run_pass("full")
            h = self.head["full"]
            fb = False
        else:
            self.run_pass("little")
            h = self.head["little"]
            if forced_fallback is None:
                with torch.cuda.stream(self.stream):
                    fb = bool(h["fallback"].item())
            else:
                self.stream.synchronize()
                fb = bool(forced_fallback)
            if rt:
                N.lib.mobile_offload_sync(rt.h)
            if fb:
                self.run_pass("big")
                h = self.head["big"]
        with torch.cuda.stream(self.stream):
            if next_token is None:  # greedy feedback on the device
                K.advance(self.pos, self.tok, h["argmax"])
            else:  # teacher-forced input stream (synthetic token ids from the host)
                K.advance(self.pos)
                self.tok_host[0] = next_token
                K.memcpy_async(self.tok, self.tok_host)
            token = int(h["argmax"].item())
        if rt:
            rt.token_end()
        return token, fb

    def decode(self, prompt: list[int], n_tokens: int, fallback_flags=None, inputs: list[int] | None = None,
               prefill_k: int | None = None, full: bool = False):
        """Public decode call: prefill `prompt`, then `n_tokens` MoBiLE steps.
        `inputs` (optional) teacher-forces the next input ids (synthetic
        streams); otherwise greedy feedback.  Returns (tokens, fallbacks)."""
        self.prefill(prompt, prefill_k)
        out, fbs = [], 0
        for i in range(n_tokens):
            forced = None if fallback_flags is None else bool(fallback_flags[i])
            nxt = None if inputs is None else int(inputs[i])
            tok, fb = self.step(forced, full=full, next_token=nxt)
            out.append(tok)
            fbs += fb
        return out, fbs
