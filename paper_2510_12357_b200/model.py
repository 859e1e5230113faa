"""Device model: the MoBiLE MoE layer (carved out of toymoe.py:188-207) plus
the surrounding decoder (attention, head) that feeds it.

`MoBiLEMoE.forward` is the hot path: fused router/top-k/replay (libmobile
router kernel) -> deterministic permute -> grouped expert GEMVs (gate-up,
down) -> shared experts -> weighted combine + residual.  Attention, embedding
and the KV cache are plumbing done with torch tensor ops on the device
(attention is out of scope for custom kernels).

Two execution modes share these kernels:
  * recompute (`forward_recompute`): the reference's semantics -- the whole
    sequence is recomputed at the pass width, replay only at the final
    position (toymoe.py:143-210).  Used by the drop-in `forward`/`generate`.
  * KV-cached decode (`DecodeSession`): one position per step; a position's
    K/V come from the pass whose output was accepted (big overwrites).
"""

from __future__ import annotations

import math
import os

import numpy as np
import torch
import torch.nn.functional as Fn

from . import _native as N
from . import kernels as K
from .spec import ModelSpec
from .weights import DeviceWeights

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False

_ACT = {"relu": N.ACT_RELU, "swiglu": N.ACT_SWIGLU}
# expert FFN implementation: "stream" (bulk-copy TMA streaming, default) or
# "warp" (register-streaming warp kernels); both are libmobile sm_100a kernels
FFN_IMPL = os.environ.get("MOBILE_FFN", "stream")  # "stream_only": never the tcgen05 path (tests)
# prefill / batched (T > TC_MIN_TOKENS): grouped expert GEMM on tcgen05 tensor cores
TC_MIN_TOKENS = int(os.environ.get("MOBILE_TC_MIN_TOKENS", "5"))
_GATE = {"selected_softmax": N.GATE_SELECTED_SOFTMAX, "softmax_all": N.GATE_SOFTMAX_ALL}


def positional(n: int, d: int, start: int, device) -> torch.Tensor:
    """Sinusoidal encoding, toymoe.py:135-140 (computed in fp64, stored f32)."""
    pos = torch.arange(start, start + n, device=device, dtype=torch.float64)[:, None]
    dim = torch.arange(d, device=device, dtype=torch.float64)[None, :]
    angle = pos / torch.pow(10000.0, (2 * (dim // 2)) / d)  # scalar base: no host copy (graph-capturable)
    return torch.where(dim.long() % 2 == 0, torch.sin(angle), torch.cos(angle)).to(torch.float32)


def pos_rows(spec: ModelSpec, n: int, start: int, device) -> torch.Tensor:
    """Positional rows added to the embeddings (zeros for pos_encoding="none")."""
    if spec.pos_encoding == "none":
        return torch.zeros(n, spec.hidden_dim, device=device, dtype=torch.float32)
    return positional(n, spec.hidden_dim, start, device)


class ExpertLocation:
    """Where a layer's routed experts live: resident tensor or cache slot pool
    (`n_slots` = experts addressable from the base, for TMA maps)."""

    def __init__(self, w13_base: int, w2_base: int, stride: int, slot: torch.Tensor | None, n_slots: int = 0):
        self.w13_base, self.w2_base, self.stride, self.slot = w13_base, w2_base, stride, slot
        self.n_slots = n_slots


class MoBiLEMoE:
    """The MoBiLE MoE layer on the device (all layers of one model)."""

    def __init__(self, dw: DeviceWeights):
        self.dw = dw
        s = dw.spec
        self.spec = s
        self.E, self.d, self.I = s.num_experts, s.hidden_dim, s.ffn
        self.S, self.Is = s.n_shared, s.shared_ffn
        self.wcode = K.dtype_code(torch.empty(0, dtype=dw.wdtype))
        self.act = _ACT[s.activation]
        self.gate_norm = _GATE[s.gate_norm]
        self._scratch: dict = {}

    def resident(self, layer: int) -> ExpertLocation:
        dw = self.dw
        base = dw.experts[layer].data_ptr()
        return ExpertLocation(base, base + dw.w13_elems * dw.elem_bytes, dw.expert_bytes, None, self.E)

    def scratch(self, T: int, k_max: int) -> dict:
        key = (T, k_max)
        sc = self._scratch.get(key)
        if sc is not None:
            return sc
        dev, E, d = self.dw.device, self.E, self.d
        f32, i32 = torch.float32, torch.int32
        ne = max(self.dw.n_gate_rows, 1)
        sc = dict(
            router=dict(h2=torch.empty(T, d, device=dev, dtype=f32), logits=torch.empty(T, E, device=dev, dtype=f32),
                        extra=torch.empty(T, ne, device=dev, dtype=f32), idx=torch.empty(T, k_max, device=dev, dtype=i32),
                        gates=torch.empty(T, k_max, device=dev, dtype=f32), flags=torch.zeros(1, device=dev, dtype=i32)),
            perm=dict(offsets=torch.empty(E + 1, device=dev, dtype=i32),
                      sorted_pairs=torch.zeros(T * k_max, device=dev, dtype=i32),  # tail stays a valid index
                      active=torch.empty(E + 1, device=dev, dtype=i32)),
            U=torch.empty(T * k_max, self.I, device=dev, dtype=f32),
            Y=torch.empty(T * k_max, d, device=dev, dtype=f32),
            x_out=torch.empty(T, d, device=dev, dtype=f32),
        )
        if self.S:
            S = self.S
            sc["s_offsets"] = torch.arange(0, (S + 1) * T, T, device=dev, dtype=i32)
            # expert s's pairs are t*S + s for t = 0..T-1 (token-major)
            sc["s_pairs"] = (torch.arange(T, device=dev, dtype=i32)[None, :] * S +
                             torch.arange(S, device=dev, dtype=i32)[:, None]).reshape(-1).contiguous()
            sc["s_active"] = torch.cat([torch.tensor([S], dtype=i32), torch.arange(S, dtype=i32)]).to(dev)
            sc["Us"] = torch.empty(T * S, self.Is, device=dev, dtype=f32)
            sc["Ys"] = torch.empty(T * S, d, device=dev, dtype=f32)
        self._scratch[key] = sc
        return sc

    def route(self, x: torch.Tensor, layer: int, k_tok: torch.Tensor, k_max: int, *, replay=None,
              replay_mask=None, reuse_gates=False, logits_out=None, idx_out=None,
              prefetch_experts: bool = False) -> dict:
        """Router + permute (toymoe.py:188-201): returns the scratch dict with
        `router` (h2, logits, idx, gates, ...) and `perm` (offsets, pairs, active).
        prefetch_experts (resident experts, decode): the router launch moves
        the selected experts' gate-up weights toward L2 once it knows them."""
        T = x.shape[0]
        sc = self.scratch(T, k_max)
        rout = sc["router"]
        if logits_out is not None or idx_out is not None:
            rout = dict(rout)
            if logits_out is not None:
                rout["logits"] = logits_out
            if idx_out is not None:
                rout["idx"] = idx_out
        pf = None
        if prefetch_experts:
            loc = self.resident(layer)
            pf = (loc.w13_base, loc.stride, self.dw.w13_elems * self.dw.elem_bytes)
        r = K.router_topk(x, self.dw.router[layer], self.E, k_max, k_tok, n_extra=self.dw.n_gate_rows,
                          replay=replay, replay_mask=replay_mask, reuse_gates=reuse_gates,
                          gate_norm=self.gate_norm, out=rout, perm=sc["perm"], prefetch=pf)
        return dict(sc, router=r)

    def experts(self, x: torch.Tensor, layer: int, sc: dict, k_tok: torch.Tensor, k_max: int,
                loc: ExpertLocation | None = None, timer=None, ln_out=None, x_out=None,
                shared_join=None) -> torch.Tensor:
        """Grouped expert FFN + shared experts + combine/residual (toymoe.py:202-207).

        Decode (T < TC_MIN_TOKENS): bulk-copy streaming GEMV launches (gate-up
        of routed + shared experts in one launch, then down of both) and the
        combine.  Prefill / batched: the tcgen05 grouped GEMM.  `shared_join`
        (batched engine): the shared experts were launched from the residual
        by shared_from_residual on a side stream; called before the combine
        (it makes the current stream wait for them).
        FFN_IMPL="stream_only" keeps the streaming path for any T (tests)."""
        T = x.shape[0]
        loc = loc if loc is not None else self.resident(layer)
        r = sc["router"]
        if T >= TC_MIN_TOKENS and self.tc_ok and FFN_IMPL != "stream_only":
            self._routed_tc(r["h2"], sc["perm"], T, k_max, loc, sc)
            if shared_join is not None:  # shared experts already running on a side stream
                shared_join()
                Ys = sc["Ys"]
            else:
                Ys = self._shared_tc(r["h2"], layer, T, sc) if self.S else None
        else:
            self._stream_ffn(r["h2"], sc["perm"], layer, T, k_max, loc, sc, timer)
            Ys = sc["Ys"] if self.S else None
        shared_logits = r["extra"] if self.dw.n_gate_rows else None
        out = sc["x_out"] if x_out is None else x_out
        K.combine(x, sc["Y"], r["gates"], k_tok, Ys, self.S, shared_logits, x_out=out, ln_out=ln_out)
        return out

    def _stream_ffn(self, h2, p, layer, T, k_max, loc, sc, timer=None, shared=True):
        """Decode FFN on the bulk-copy engine: writes sc["Y"] (and sc["Ys"])."""
        dw, E, d = self.dw, self.E, self.d
        max_active = min(E, T * k_max)
        act_epi = K.EPI_SWIGLU if self.act == N.ACT_SWIGLU else K.EPI_RELU
        rows13 = 2 * self.I if self.act == N.ACT_SWIGLU else self.I
        g_up = [K.sg_group(w_base=loc.w13_base, stride=loc.stride, slot=loc.slot, K=d, rows=rows13, x=h2,
                           x_div=k_max, offsets=p["offsets"], pairs=p["sorted_pairs"], active=p["active"],
                           max_active=max_active, out=sc["U"], epi=act_epi)]
        g_dn = [K.sg_group(w_base=loc.w2_base, stride=loc.stride, slot=loc.slot, K=self.I, rows=d, x=sc["U"],
                           offsets=p["offsets"], pairs=p["sorted_pairs"], active=p["active"],
                           max_active=max_active, out=sc["Y"])]
        if self.S and shared:
            base, sb = dw.shared[layer].data_ptr(), dw.shared_bytes
            rows13s = 2 * self.Is if self.act == N.ACT_SWIGLU else self.Is
            # shared experts first: their weights and (constant) pair lists are
            # static, so their copies start before the PDL wait on the router
            g_up.insert(0, K.sg_group(w_base=base, stride=sb, K=d, rows=rows13s, x=h2, x_div=self.S,
                                      offsets=sc["s_offsets"], pairs=sc["s_pairs"], active=sc["s_active"],
                                      max_active=self.S, out=sc["Us"], epi=act_epi, prefetch=True))
            g_dn.insert(0, K.sg_group(w_base=base + dw.s_w13_elems * dw.elem_bytes, stride=sb, K=self.Is, rows=d,
                                      x=sc["Us"], offsets=sc["s_offsets"], pairs=sc["s_pairs"],
                                      active=sc["s_active"], max_active=self.S, out=sc["Ys"], prefetch=True))
        if timer is not None:
            timer.start()
        K.stream_gemv(g_up, self.wcode, T)
        if timer is not None:
            timer.stop(("gate_up", T, k_max))
        K.stream_gemv(g_dn, self.wcode, T)

    @property
    def tc_ok(self) -> bool:
        """Shapes/dtype the tcgen05 grouped GEMM supports (bf16, K % 64, N % 128)."""
        d, I, Is = self.d, self.I, self.Is
        return (self.dw.wdtype == torch.bfloat16 and self.act == N.ACT_SWIGLU and d % 128 == 0
                and I % 64 == 0 and (2 * I) % 128 == 0 and (not self.S or (Is % 64 == 0 and (2 * Is) % 128 == 0)))

    def _tc_scratch(self, sc: dict, T: int, k_max: int) -> dict:
        key = (T, k_max)
        tc = self._scratch[key].get("tc")
        if tc is None:
            dev, d = self.dw.device, self.d
            P = T * k_max
            bf = torch.bfloat16
            tc = dict(X=torch.empty(P, d, device=dev, dtype=bf), U=torch.empty(P, self.I, device=dev, dtype=bf))
            if self.S:
                # expert-major rows s*T + t of every shared expert (one grouped launch for all S)
                tc["Xs"] = torch.empty(self.S * T, d, device=dev, dtype=bf)
                tc["Us"] = torch.empty(self.S * T, self.Is, device=dev, dtype=bf)
            self._scratch[key]["tc"] = tc
        return tc

    def _routed_tc(self, h2, p, T, k_max, loc, sc):
        """Routed experts on tcgen05: gather -> gate-up (SwiGLU) -> down (scatter to pairs) into sc["Y"]."""
        E, d, I = self.E, self.d, self.I
        tc = self._tc_scratch(sc, T, k_max)
        P = T * k_max
        bound = (P + 127) // 128 + min(E, P)
        n_slots = loc.n_slots or E
        K.gather_bf16(h2, p["sorted_pairs"], k_max, P, tc["X"])
        K.grouped_gemm(tc["X"], d, loc.w13_base, loc.stride, n_slots, 2 * I, offsets=p["offsets"], active=p["active"],
                       slot=loc.slot, max_tiles=bound * (2 * I // 128), epi=K.GG_SWIGLU_BF16, out_bf16=tc["U"], ldo=I)
        K.grouped_gemm(tc["U"], I, loc.w2_base, loc.stride, n_slots, d, offsets=p["offsets"], active=p["active"],
                       slot=loc.slot, max_tiles=bound * (d // 128), epi=K.GG_STORE_F32, out_f32=sc["Y"], ldo=d,
                       row_to_pair=p["sorted_pairs"])

    def shared_from_residual(self, x: torch.Tensor, layer: int, T: int, k_max: int) -> None:
        """Shared experts of a batch straight from the post-attention residual
        x: LN + bf16 gather (bit-identical to bf16 of the router's h2) and the
        two grouped launches into the (T, k_max) scratch's Ys.  They do not
        depend on the routing, so the batched engine runs them on a side
        stream concurrently with the router / permute / routed experts."""
        sc = self.scratch(T, k_max)
        tc = self._tc_scratch(sc, T, k_max)
        K.gather_ln_bf16(x, sc["s_pairs"], self.S, self.S * T, tc["Xs"])
        self._shared_gemms(layer, T, sc, tc)

    def _shared_tc(self, h2, layer, T, sc):
        """Shared experts on tcgen05 into sc["Ys"] (T, S, d): ONE grouped
        gate-up and ONE down launch for all S shared experts (expert s owns
        the rows s*T .. s*T+T-1 of a gathered copy of h2), so the S weight
        streams share the SMs instead of running S small launches in turn."""
        dw, d, Is, S = self.dw, self.d, self.Is, self.S
        tc = self._tc_scratch(sc, T, sc["perm"]["sorted_pairs"].numel() // max(T, 1))
        K.gather_bf16(h2, sc["s_pairs"], S, S * T, tc["Xs"])
        self._shared_gemms(layer, T, sc, tc)
        return sc["Ys"]

    def _shared_gemms(self, layer, T, sc, tc):
        dw, d, Is, S = self.dw, self.d, self.Is, self.S
        base = dw.shared[layer].data_ptr()
        bound = S * ((T + 127) // 128)
        K.grouped_gemm(tc["Xs"], d, base, dw.shared_bytes, S, 2 * Is, offsets=sc["s_offsets"], active=sc["s_active"],
                       max_tiles=bound * (2 * Is // 128), epi=K.GG_SWIGLU_BF16, out_bf16=tc["Us"], ldo=Is)
        K.grouped_gemm(tc["Us"], Is, base + dw.s_w13_elems * dw.elem_bytes, dw.shared_bytes, S, d,
                       offsets=sc["s_offsets"], active=sc["s_active"], max_tiles=bound * (d // 128),
                       epi=K.GG_STORE_F32, out_f32=sc["Ys"], ldo=d, row_to_pair=sc["s_pairs"])

    # ---- expert-parallel helpers (ep.py) ----
    def rows_ffn(self, layer: int, rows: torch.Tensor, ids: torch.Tensor, k_tok: torch.Tensor | None = None,
                 clone: bool = True, force_tc: bool = False, loc: ExpertLocation | None = None) -> torch.Tensor:
        """Routed-expert FFN of R independent rows, row i through local expert
        ids[i] (k = 1); rows with k_tok[i] = 0 are skipped (their output rows
        are left as they were).  force_tc: the tcgen05 path for any R (each
        output row then depends only on its input row: expert-parallel owners
        use it so the layer output does not depend on how rows are spread)."""
        R = rows.shape[0]
        if k_tok is None:
            k_tok = torch.ones(R, dtype=torch.int32, device=rows.device)
        sc = self.scratch(R, 1)
        p = K.permute(ids.view(R, 1), k_tok, self.E, out=sc["perm"])
        loc = loc if loc is not None else self.resident(layer)  # offloaded shards: the cache's slot table
        if rows.dtype == torch.bfloat16 and not self.tc_ok:
            raise ValueError("rows_ffn: bf16 rows need the tcgen05 expert path (bf16 SwiGLU shapes)")
        if (R >= TC_MIN_TOKENS or force_tc or rows.dtype == torch.bfloat16) and self.tc_ok:
            self._routed_tc(rows, p, R, 1, loc, sc)
        else:
            self._stream_ffn(rows, p, layer, R, 1, loc, sc, shared=False)
        return sc["Y"][:R].clone() if clone else sc["Y"][:R]

    def shared_rows(self, layer: int, h2: torch.Tensor, sc: dict) -> torch.Tensor:
        """Shared-expert outputs (T, S, d) for the tokens of a routed scratch."""
        T = h2.shape[0]
        k_max = sc["perm"]["sorted_pairs"].numel() // max(T, 1)
        if T >= TC_MIN_TOKENS and self.tc_ok:
            return self._shared_tc(h2, layer, T, sc)
        dw, d = self.dw, self.d
        act_epi = K.EPI_SWIGLU if self.act == N.ACT_SWIGLU else K.EPI_RELU
        base, sb = dw.shared[layer].data_ptr(), dw.shared_bytes
        rows13s = 2 * self.Is if self.act == N.ACT_SWIGLU else self.Is
        K.stream_gemv([K.sg_group(w_base=base, stride=sb, K=d, rows=rows13s, x=h2, x_div=self.S,
                                  offsets=sc["s_offsets"], pairs=sc["s_pairs"], active=sc["s_active"],
                                  max_active=self.S, out=sc["Us"], epi=act_epi, prefetch=True)], self.wcode, T)
        K.stream_gemv([K.sg_group(w_base=base + dw.s_w13_elems * dw.elem_bytes, stride=sb, K=self.Is, rows=d,
                                  x=sc["Us"], offsets=sc["s_offsets"], pairs=sc["s_pairs"], active=sc["s_active"],
                                  max_active=self.S, out=sc["Ys"], prefetch=True)], self.wcode, T)
        del k_max
        return sc["Ys"]

    def forward(self, x: torch.Tensor, layer: int, k_tok: torch.Tensor, k_max: int, *, replay=None,
                replay_mask=None, reuse_gates=False, experts: ExpertLocation | None = None,
                hook=None, timer=None, x_out=None):
        """x (T, d) f32 residual -> (x_out, scratch): route, then experts.

        `hook` (optional) has `pre(layer, router_out, perm) -> ExpertLocation`,
        run between routing and the expert kernels (the offload runtime makes
        the selected experts resident there: engine.py:137-149), and
        `post(layer)`, run once the layer's kernels are enqueued (unpin +
        last-use events: engine.py:152-153).  `timer` (optional) brackets the
        gate-up launches with CUDA events for the live roofline."""
        sc = self.route(x, layer, k_tok, k_max, replay=replay, replay_mask=replay_mask, reuse_gates=reuse_gates)
        if hook is not None:
            experts = hook.pre(layer, sc["router"], sc["perm"])
        x_out = self.experts(x, layer, sc, k_tok, k_max, experts, timer, x_out=x_out)
        if hook is not None:
            hook.post(layer)
        return x_out, sc


class DeviceModel:
    """Decoder around the MoBiLE layer (recompute and KV-cached modes)."""

    def __init__(self, dw: DeviceWeights):
        self.dw = dw
        self.spec: ModelSpec = dw.spec
        self.moe = MoBiLEMoE(dw)
        self.device = dw.device
        self.head_ws: dict = {}

    # ------------------------------------------------------------- pieces
    def _lin(self, h: torch.Tensor, w: torch.Tensor, resid: torch.Tensor | None = None,
             resid_inplace: bool = False) -> torch.Tensor:
        """(resid +) h @ w.T for an out-major weight (N, d), on libmobile kernels:
        up to 8 rows the bulk-copy GEMV (f32 activations); more rows of a bf16
        model the tcgen05 grouped GEMM in dense mode (bf16 operands, f32
        accumulate, the residual accumulated in its epilogue).  Only the f32
        toy weights (the reference-parity configs) with more than 8 rows use
        torch's matmul."""
        w = self.dw.plain(w)
        n, d = h.shape
        n_out = w.shape[0]
        if n <= 8:
            return K.dense_gemv(h.contiguous(), w, residual=resid)
        if w.dtype == torch.bfloat16 and d % 128 == 0 and n_out % 128 == 0:
            xb = torch.empty(n, d, dtype=torch.bfloat16, device=h.device)
            K.gather_bf16(h.contiguous(), None, 1, n, xb)
            if resid is not None:  # accumulated in the GEMM epilogue (in place when the caller allows)
                out, epi = (resid if resid_inplace else resid.clone()), K.GG_ACCUM_F32
            else:
                out, epi = torch.empty(n, n_out, dtype=torch.float32, device=h.device), K.GG_STORE_F32
            K.grouped_gemm(xb, d, w.data_ptr(), w.numel() * w.element_size(), 1, n_out,
                           max_tiles=(n + 127) // 128 * (n_out // 128), dense_rows=n, dense_experts=1, epi=epi,
                           out_f32=out, ldo=n_out)
            return out
        y = Fn.linear(h, w) if w.dtype == torch.float32 else Fn.linear(h.to(w.dtype), w).to(torch.float32)
        return y if resid is None else resid + y

    def attention_full(self, x: torch.Tensor, layer: int) -> torch.Tensor:
        """toymoe.py:178-186 over all n positions (causal), n_heads generalised."""
        dw, s = self.dw, self.spec
        n, d = x.shape
        h = Fn.layer_norm(x, (d,), eps=1e-5)
        kvd = s.kv_dim
        q, k, v = self._lin(h, dw.qkv[layer]).split([d, kvd, kvd], dim=-1)
        H, Hk = s.n_heads, s.kv_heads
        hd = d // H
        qh = q.reshape(n, H, hd).transpose(0, 1)
        # grouped-query attention: query head h reads key/value head h // (H / Hk)
        kh, vh = (t.reshape(n, Hk, hd).transpose(0, 1).repeat_interleave(H // Hk, dim=0) for t in (k, v))
        scores = (qh @ kh.transpose(1, 2)) / math.sqrt(hd)
        mask = torch.ones(n, n, dtype=torch.bool, device=x.device).triu(1)
        scores = scores.masked_fill(mask, float("-inf"))
        attn = torch.softmax(scores, dim=-1)
        out = (attn @ vh).transpose(0, 1).reshape(n, d)
        return self._lin(out, dw.o[layer], resid=x)

    def stream_head_ws(self) -> K.StreamHeadWorkspace:
        if getattr(self, "_sh_ws", None) is None:
            self._sh_ws = K.StreamHeadWorkspace(self.device)
        return self._sh_ws

    def head_workspace(self, T: int) -> K.HeadWorkspace:
        ws = self.head_ws.get(T)
        if ws is None:
            ws = self.head_ws[T] = K.HeadWorkspace(T, self.spec.vocab_size, self.device)
        return ws

    # ------------------------------------------------------------- recompute
    def forward_recompute(self, tokens, k: int, replay_states=None, reuse_gates=False):
        """toymoe.forward on the device.  Returns device tensors
        (probs f64 (V,), states f32 (L, E), selections int32 (L, k), flags)."""
        s, dw = self.spec, self.dw
        dev = self.device
        n = len(tokens)
        tok = torch.as_tensor(np.asarray(tokens, dtype=np.int64)).to(dev)
        x = dw.embed[tok] + pos_rows(s, n, 0, dev)
        k_tok = torch.full((n,), k, dtype=torch.int32, device=dev)
        replay = mask = None
        if replay_states is not None:
            rs = torch.as_tensor(np.asarray(replay_states, dtype=np.float32)).to(dev)
            replay = torch.zeros(n, s.num_experts, device=dev, dtype=torch.float32)
            mask = torch.zeros(n, device=dev, dtype=torch.uint8)
            mask[-1] = 1
        states = torch.empty(s.num_layers, s.num_experts, device=dev, dtype=torch.float32)
        sels = torch.empty(s.num_layers, k, device=dev, dtype=torch.int32)
        flags = torch.zeros(1, device=dev, dtype=torch.int32)
        for layer in range(s.num_layers):
            x = self.attention_full(x, layer)
            if replay is not None:
                replay[-1] = rs[layer]
            x_new, sc = self.moe.forward(x, layer, k_tok, k, replay=replay, replay_mask=mask, reuse_gates=reuse_gates)
            states[layer] = sc["router"]["logits"][-1]
            sels[layer] = sc["router"]["idx"][-1]
            flags |= sc["router"]["flags"]
            sc["router"]["flags"].zero_()
            x = x_new.clone()
        logits = torch.empty(1, s.vocab_size, device=dev, dtype=torch.float32)
        x_ln = Fn.layer_norm(x[-1:], (s.hidden_dim,), eps=1e-5).contiguous()
        K.stream_head(x_ln, dw.head, 0.0, s.logit_scale, ws=self.stream_head_ws(), logits_out=logits)
        probs = K.softmax_rows(logits, torch.float64)[0]
        return probs, states, sels, flags


class DecodeSession:
    """KV-cached decode for B sequences at a common position."""

    def __init__(self, model: DeviceModel, batch: int, max_len: int):
        s = model.spec
        self.m, self.B, self.max_len = model, batch, max_len
        dev = model.device
        # head-major KV cache (L, B, Hkv, max_len, head_dim): one key/value
        # head's positions are contiguous, so a (head, position-chunk) block is
        # one bulk copy (Hkv = kv_heads: fewer than the query heads under GQA)
        self.kc = torch.zeros(s.num_layers, batch, s.kv_heads, max_len, s.hidden_dim // s.n_heads, device=dev,
                              dtype=torch.float32)
        self.vc = torch.zeros_like(self.kc)
        self.pos = 0
        self.moe_forward = None  # optional MoE layer override (expert parallelism: ep.EPStepEngine.prefill)

    def _attn_step(self, x: torch.Tensor, layer: int, rows: torch.Tensor | None, pos: int, n: int):
        """Attention for n new positions [pos, pos+n) of the sequences `rows`
        (None = all); writes their K/V into the cache."""
        m, s = self.m, self.m.spec
        dw = m.dw
        Bn = x.shape[0] // n
        d = s.hidden_dim
        H, Hk, kvd = s.n_heads, s.kv_heads, s.kv_dim
        hd = d // H
        h = Fn.layer_norm(x, (d,), eps=1e-5)
        qkv = m._lin(h, dw.qkv[layer])
        q, k, v = qkv.split([d, kvd, kvd], dim=-1)
        q = q.reshape(Bn, n, d)
        kn = k.reshape(Bn, n, Hk, hd).transpose(1, 2)
        vn = v.reshape(Bn, n, Hk, hd).transpose(1, 2)
        if rows is None:
            self.kc[layer, :, :, pos:pos + n] = kn
            self.vc[layer, :, :, pos:pos + n] = vn
            kh, vh = self.kc[layer, :, :, :pos + n], self.vc[layer, :, :, :pos + n]
        else:
            self.kc[layer, rows, :, pos:pos + n] = kn
            self.vc[layer, rows, :, pos:pos + n] = vn
            kh, vh = self.kc[layer, rows, :, :pos + n], self.vc[layer, rows, :, :pos + n]
        qh = q.view(Bn, n, H, hd).transpose(1, 2)
        if n > 1:
            # prompt chunk: fused attention (torch SDPA: flash on bf16 operands
            # for bf16 models -- f32 accumulate, the weights' precision already
            # bounds the error -- memory-efficient f32 otherwise), causal with
            # the chunk's offset into the cache
            dt = torch.bfloat16 if dw.wdtype == torch.bfloat16 else torch.float32
            if pos == 0 and rows is None:  # the whole context is this chunk: one conversion of the qkv rows
                qkv_t = qkv.to(dt).view(Bn, n, d + 2 * kvd)
                qs = qkv_t[..., :d].view(Bn, n, H, hd).transpose(1, 2)
                ks = qkv_t[..., d:d + kvd].view(Bn, n, Hk, hd).transpose(1, 2)
                vs = qkv_t[..., d + kvd:].view(Bn, n, Hk, hd).transpose(1, 2)
                out = Fn.scaled_dot_product_attention(qs, ks, vs, is_causal=True, enable_gqa=Hk != H)
            else:
                mask = torch.ones(n, pos + n, dtype=torch.bool, device=x.device).tril(pos)
                out = Fn.scaled_dot_product_attention(qh.to(dt), kh.to(dt), vh.to(dt), attn_mask=mask,
                                                      enable_gqa=Hk != H)
            out = out.float().transpose(1, 2).reshape(Bn * n, d)
            return m._lin(out, dw.o[layer], resid=x, resid_inplace=True)
        if Hk != H:
            kh, vh = kh.repeat_interleave(H // Hk, dim=1), vh.repeat_interleave(H // Hk, dim=1)
        scores = (qh @ kh.transpose(-1, -2)) / math.sqrt(hd)
        attn = torch.softmax(scores, dim=-1)
        out = (attn @ vh).transpose(1, 2).reshape(Bn * n, d)
        return m._lin(out, dw.o[layer], resid=x)

    def run(self, tokens: torch.Tensor, k_tok: torch.Tensor, k_max: int, *, rows=None, replay=None,
            replay_mask=None, reuse_gates=False, advance=True, expert_hook=None, layer_hook=None, timer=None):
        """Process `tokens` (Bn, n) at positions [pos, pos+n).  Returns
        (x_last (Bn, d), states (L, Bn*n, E) view of last-position logits, idx (L, Bn, k_max)).
        `replay` (L, Bn, E) applies to the last position of every row with replay_mask."""
        m, s = self.m, self.m.spec
        dw, dev = m.dw, m.device
        Bn, n = tokens.shape
        pos = self.pos
        x = dw.embed[tokens.reshape(-1)] + pos_rows(s, n, pos, dev).repeat(Bn, 1)
        T = Bn * n
        states = torch.empty(s.num_layers, Bn, s.num_experts, device=dev, dtype=torch.float32)
        idx = torch.empty(s.num_layers, Bn, k_max, device=dev, dtype=torch.int32)
        rep_full = rep_mask_full = None
        if replay is not None:
            rep_full = torch.zeros(T, s.num_experts, device=dev, dtype=torch.float32)
            rep_mask_full = torch.zeros(T, device=dev, dtype=torch.uint8)
            last = torch.arange(Bn, device=dev) * n + (n - 1)
            rep_mask_full[last] = replay_mask if replay_mask is not None else 1
        spare = None  # the residual buffer the next combine writes
        for layer in range(s.num_layers):
            if layer_hook is not None:
                layer_hook(layer)
            x = self._attn_step(x, layer, rows, pos, n)
            if replay is not None:
                rep_full[last] = replay[layer]
            if self.moe_forward is not None:  # expert-parallel layer (ep.py): (x_new, scratch)
                x_new, sc = self.moe_forward(x, layer, k_tok, k_max, replay=rep_full, replay_mask=rep_mask_full,
                                             reuse_gates=reuse_gates)
                x_new = x_new.clone()
            else:  # the combine writes the other of two residual buffers (no copy per layer)
                if spare is None:
                    spare = torch.empty_like(x)
                x_new, sc = m.moe.forward(x, layer, k_tok, k_max, replay=rep_full, replay_mask=rep_mask_full,
                                          reuse_gates=reuse_gates, hook=expert_hook, timer=timer, x_out=spare)
                spare = x
            lg = sc["router"]["logits"].view(Bn, n, s.num_experts)
            states[layer] = lg[:, -1]
            idx[layer] = sc["router"]["idx"].view(Bn, n, k_max)[:, -1]
            x = x_new
        if advance:
            self.pos += n
        x_last = x.view(Bn, n, s.hidden_dim)[:, -1].contiguous()
        return x_last, states, idx
