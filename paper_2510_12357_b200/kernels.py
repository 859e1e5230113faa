"""Thin torch-tensor wrappers over the libmobile C ABI.

Tensors must already live on the CUDA device (the C ABI takes raw pointers);
every call is enqueued on the current torch stream unless `stream` is given.
"""

from __future__ import annotations

import torch

from . import _native as N

_DT = {torch.float32: N.F32, torch.bfloat16: N.BF16, torch.float64: N.F64}

# number of libmobile kernel launches issued through these wrappers (bench's gpu_launches)
LAUNCHES = [0]


def _count(n: int = 1) -> None:
    LAUNCHES[0] += n


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise N.MobileNativeError(f"unsupported dtype {t.dtype}") from None


def _s(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise N.MobileNativeError("libmobile kernels take CUDA tensors only (no CPU fallback)")


def router_topk(x, w_router, E, k_max, k_tok, *, n_extra=0, replay=None, replay_mask=None,
                reuse_gates=False, gate_norm=N.GATE_SELECTED_SOFTMAX, out=None, perm=None, stream=None,
                prefetch=None):
    """Fused LN + router GEMV + top-k + replay + gates (toymoe.py:188-201).
    With `perm` (dict offsets/sorted_pairs/active) the permute is fused too.
    `prefetch` = (base, stride, bytes): the selected experts' first bytes go
    toward L2 once the selection is known (no result changes)."""
    _dev(x, w_router, k_tok, replay, replay_mask)
    T, d = x.shape
    dev = x.device
    if out is None:
        out = dict(
            h2=torch.empty(T, d, device=dev, dtype=torch.float32),
            logits=torch.empty(T, E, device=dev, dtype=torch.float32),
            extra=torch.empty(T, max(n_extra, 1), device=dev, dtype=torch.float32),
            idx=torch.empty(T, k_max, device=dev, dtype=torch.int32),
            gates=torch.empty(T, k_max, device=dev, dtype=torch.float32),
            flags=torch.zeros(1, device=dev, dtype=torch.int32),
        )
    pf_base, pf_stride, pf_bytes = prefetch if prefetch is not None else (None, 0, 0)
    st = N.lib.mobile_router_topk_pf(
        N.ptr(x), N.ptr(out["h2"]), N.ptr(w_router), dtype_code(w_router), T, d, E, n_extra, k_max,
        N.ptr(k_tok), N.ptr(replay), N.ptr(replay_mask), int(bool(reuse_gates)), gate_norm,
        N.ptr(out["logits"]), N.ptr(out["extra"]) if n_extra else None, N.ptr(out["idx"]),
        N.ptr(out["gates"]), N.ptr(out["flags"]),
        N.ptr(perm["offsets"]) if perm else None, N.ptr(perm["sorted_pairs"]) if perm else None,
        N.ptr(perm["active"]) if perm else None, pf_base, int(pf_stride), int(pf_bytes), _s(stream))
    _count()
    N.check(st, "router_topk")
    return out


def topk_rows(rows: torch.Tensor, k: int, stream=None):
    """Stable top-k per row (toymoe.py:80-88) -> (idx (R,k) int32, flags (1,) int32)."""
    _dev(rows)
    rows = rows.contiguous()
    R, E = rows.shape
    idx = torch.empty(R, max(k, 0), device=rows.device, dtype=torch.int32)
    flags = torch.zeros(1, device=rows.device, dtype=torch.int32)
    _count()
    N.check(N.lib.mobile_topk_rows(N.ptr(rows), dtype_code(rows), R, E, k, N.ptr(idx), N.ptr(flags), _s(stream)),
            "topk_rows")
    return idx, flags


class HeadWorkspace:
    def __init__(self, T: int, V: int, device):
        n = int(N.lib.mobile_head_ws_bytes(T, V))
        self.buf = torch.zeros(n, dtype=torch.uint8, device=device)  # ticket words start (and stay) 0
        self.T, self.V = T, V


def head_confidence(x, w_head, gamma, logit_scale, *, ws: HeadWorkspace, logits_out=None, out=None,
                    stream=None):
    """conf = max softmax(LN(x) @ head * scale), first argmax, fallback = conf <= gamma."""
    _dev(x, w_head)
    T, d = x.shape
    V = w_head.shape[0]
    if ws.T < T or ws.V != V:
        raise N.MobileNativeError("head workspace too small")
    if out is None:
        out = dict(conf=torch.empty(T, device=x.device, dtype=torch.float32),
                   argmax=torch.empty(T, device=x.device, dtype=torch.int32),
                   fallback=torch.empty(T, device=x.device, dtype=torch.uint8))
    _count()
    N.check(N.lib.mobile_head_confidence(
        N.ptr(x), N.ptr(w_head), dtype_code(w_head), T, d, V, float(logit_scale), float(gamma),
        N.ptr(logits_out), N.ptr(out["conf"]), N.ptr(out["argmax"]), N.ptr(out["fallback"]),
        N.ptr(ws.buf), _s(stream)), "head_confidence")
    return out


def softmax_rows(logits: torch.Tensor, out_dtype=torch.float64, stream=None):
    _dev(logits)
    logits = logits.contiguous()
    T, V = logits.shape
    probs = torch.empty(T, V, device=logits.device, dtype=out_dtype)
    _count()
    N.check(N.lib.mobile_softmax_rows(N.ptr(logits), dtype_code(logits), N.ptr(probs), dtype_code(probs),
                                      T, V, _s(stream)), "softmax_rows")
    return probs


def probs_check(probs: torch.Tensor, stream=None):
    """(sum, max) of a probability row in f64 (policy.py:69-79 inputs)."""
    _dev(probs)
    out = torch.empty(2, device=probs.device, dtype=torch.float64)
    _count()
    N.check(N.lib.mobile_probs_check(N.ptr(probs.contiguous()), dtype_code(probs), probs.numel(), N.ptr(out),
                                     _s(stream)), "probs_check")
    return out


def permute(idx, k_tok, E, out=None, stream=None):
    _dev(idx, k_tok)
    T, k_max = idx.shape
    dev = idx.device
    if out is None:
        out = dict(offsets=torch.empty(E + 1, device=dev, dtype=torch.int32),
                   sorted_pairs=torch.empty(max(T * k_max, 1), device=dev, dtype=torch.int32),
                   active=torch.empty(E + 1, device=dev, dtype=torch.int32))
    _count()
    N.check(N.lib.mobile_permute(N.ptr(idx), N.ptr(k_tok), T, k_max, E, N.ptr(out["offsets"]),
                                 N.ptr(out["sorted_pairs"]), N.ptr(out["active"]), _s(stream)), "permute")
    return out


def combine(x, Y, gates, k_tok, Y_shared=None, n_shared=0, shared_logits=None, x_out=None, ln_out=None,
            stream=None):
    T, d = x.shape
    k_max = gates.shape[1]
    if x_out is None:
        x_out = torch.empty_like(x)
    _count()
    N.check(N.lib.mobile_combine(N.ptr(x), N.ptr(Y), N.ptr(gates), N.ptr(k_tok), T, k_max, d, N.ptr(Y_shared),
                                 int(n_shared), N.ptr(shared_logits), N.ptr(x_out), N.ptr(ln_out), _s(stream)),
            "combine")
    return x_out


EPI_STORE, EPI_RELU, EPI_SWIGLU = 0, 1, 2


def sg_group(*, w_base: int, K: int, rows: int, x, out, epi=EPI_STORE, stride=0, slot=None, x_div=1,
             offsets=None, pairs=None, active=None, max_active=1, dense_T=0, residual=None, prefetch=None):
    """`prefetch` (default: dense groups) marks groups whose weights and expert
    lists are static, so their copies may start before the PDL wait."""
    if prefetch is None:
        prefetch = offsets is None
    return N.mobile_sg_group(w_base, int(stride), N.ptr(slot), N.ptr(x), int(x_div), N.ptr(offsets), N.ptr(pairs),
                             N.ptr(active), int(dense_T), int(max_active), int(K), int(rows), N.ptr(out),
                             N.ptr(residual), int(epi), int(bool(prefetch)))


def stream_gemv(groups, w_dtype: int, max_tokens: int, stream=None):
    """Bulk-copy streaming GEMV over 1..4 groups in one launch (mobile_stream_gemv)."""
    arr = (N.mobile_sg_group * len(groups))(*groups)
    _count()
    N.check(N.lib.mobile_stream_gemv(arr, len(groups), w_dtype, int(max_tokens), _s(stream)), "stream_gemv")


def dense_gemv(x, w, *, do_ln=False, residual=None, out=None, stream=None):
    """y = (residual +) LN?(x) @ w.T for T <= 8 rows; w (N, d) out-major."""
    _dev(x, w)
    T, d = x.shape
    n_out = w.shape[0]
    if out is None:
        out = torch.empty(T, n_out, device=x.device, dtype=torch.float32)
    _count()
    _native_check(T, d, do_ln, x, w, n_out, residual, out, stream)
    return out


def attn_split_workspace(B, d, n_heads, max_len, device):
    """Caller-owned split-KV workspace for attn_decode (decoder.cu): (partials,
    tickets) sized by mobile_attn_split_ws, or None when the shape runs unsplit.
    One per concurrently running caller (engine stream / captured graph)."""
    import ctypes
    nf, nt = ctypes.c_int(0), ctypes.c_int(0)
    N.check(N.lib.mobile_attn_split_ws(B, d, n_heads, max_len, ctypes.byref(nf), ctypes.byref(nt)), "attn_split_ws")
    if nf.value == 0:
        return None
    return (torch.empty(nf.value, dtype=torch.float32, device=device),
            torch.zeros(nt.value, dtype=torch.int32, device=device))


def attn_decode(qkv, k_cache, v_cache, pos, n_heads, out=None, stream=None, ws=None):
    """qkv (B, d + 2 Hkv hd); caches head-major (B, Hkv, max_len, hd); Hkv < n_heads = GQA."""
    B = qkv.shape[0]
    Hkv, max_len, hd = k_cache.shape[1], k_cache.shape[2], k_cache.shape[3]
    d = n_heads * hd
    if out is None:
        out = torch.empty(B, d, device=qkv.device, dtype=torch.float32)
    _count()
    wp, tp, nf, nt = (N.ptr(ws[0]), N.ptr(ws[1]), ws[0].numel(), ws[1].numel()) if ws is not None else (None, None, 0, 0)
    N.check(N.lib.mobile_attn_decode_ws(N.ptr(qkv), N.ptr(k_cache), N.ptr(v_cache), N.ptr(pos), B, d, n_heads,
                                        Hkv, max_len, N.ptr(out), wp, tp, nf, nt, _s(stream)), "attn_decode")
    return out


def embed(tok, pos, table, pe, out, ln_out=None, stream=None):
    B = tok.shape[0]
    _count()
    N.check(N.lib.mobile_embed(N.ptr(tok), N.ptr(pos), N.ptr(table), N.ptr(pe), B, table.shape[1], N.ptr(out),
                               N.ptr(ln_out), _s(stream)), "embed")
    return out


def advance(pos, tok=None, next_tok=None, stream=None):
    _count()
    N.check(N.lib.mobile_advance(N.ptr(pos), pos.shape[0], N.ptr(tok), N.ptr(next_tok), _s(stream)), "advance")


def _native_check(T, d, do_ln, x, w, n_out, residual, out, stream):
    N.check(N.lib.mobile_dense_gemv(N.ptr(x), T, d, int(bool(do_ln)), N.ptr(w), dtype_code(w), n_out,
                                    N.ptr(residual), N.ptr(out), _s(stream)), "dense_gemv")


def memcpy_async(dst: torch.Tensor, src: torch.Tensor, stream=None):
    """Raw cudaMemcpyAsync (graph-capturable) between pinned host and device tensors."""
    n = src.numel() * src.element_size()
    N.check(N.lib.mobile_memcpy_async(N.ptr(dst), N.ptr(src), n, _s(stream)), "memcpy_async")


class StreamHeadWorkspace:
    def __init__(self, device):
        self.buf = torch.zeros(int(N.lib.mobile_stream_head_ws_bytes()), dtype=torch.uint8, device=device)


def stream_head(x_ln, w_head, gamma, logit_scale, *, ws: StreamHeadWorkspace, logits_out=None, out=None,
                stream=None):
    """Head + confidence on the bulk-copy engine (x_ln = LN(x), T <= 4 rows)."""
    _dev(x_ln, w_head)
    T, d = x_ln.shape
    V = w_head.shape[0]
    if out is None:
        out = dict(conf=torch.empty(T, device=x_ln.device, dtype=torch.float32),
                   argmax=torch.empty(T, device=x_ln.device, dtype=torch.int32),
                   fallback=torch.empty(T, device=x_ln.device, dtype=torch.uint8))
    _count()
    N.check(N.lib.mobile_stream_head(N.ptr(x_ln), T, d, N.ptr(w_head), dtype_code(w_head), V, float(logit_scale),
                                     float(gamma), N.ptr(logits_out), N.ptr(out["conf"]), N.ptr(out["argmax"]),
                                     N.ptr(out["fallback"]), N.ptr(ws.buf), _s(stream)), "stream_head")
    return out


GG_STORE_F32, GG_SWIGLU_BF16, GG_STORE_BF16, GG_ACCUM_F32 = 0, 1, 2, 3


def _gg_call(A, K, B_base, b_expert_stride, n_slots, n_cols, offsets, active, slot, max_tiles, dense_rows,
             dense_experts, epi, out_f32, out_bf16, ldo, out_expert_stride, row_to_pair, stream):
    N.check(N.lib.mobile_grouped_gemm(
        N.ptr(A), A.shape[0], int(K), int(B_base), int(b_expert_stride), int(n_slots), int(n_cols), N.ptr(offsets),
        N.ptr(active), N.ptr(slot), int(max_tiles), int(dense_rows), int(dense_experts), int(epi), N.ptr(out_f32),
        N.ptr(out_bf16), int(ldo), int(out_expert_stride), N.ptr(row_to_pair), _s(stream)), "grouped_gemm")


def grouped_gemm(A, K, B_base: int, b_expert_stride: int, n_slots: int, N_: int, *, offsets=None, active=None,
                 slot=None, max_tiles: int, dense_rows=0, dense_experts=0, epi=GG_STORE_F32, out_f32=None,
                 out_bf16=None, ldo=0, out_expert_stride=0, row_to_pair=None, stream=None):
    """tcgen05 grouped GEMM (mobile_grouped_gemm)."""
    _count()
    _gg_call(A, K, B_base, b_expert_stride, n_slots, N_, offsets, active, slot, max_tiles, dense_rows, dense_experts,
             epi, out_f32, out_bf16, ldo, out_expert_stride, row_to_pair, stream)


def logits_confidence(logits, logit_scale, gamma, out, stream=None):
    """conf / argmax / fallback of raw logits rows (T, V) f32 (head GEMM output)."""
    _dev(logits)
    T, V = logits.shape
    _count()
    N.check(N.lib.mobile_logits_confidence(N.ptr(logits), T, V, float(logit_scale), float(gamma), N.ptr(out["conf"]),
                                           N.ptr(out["argmax"]), N.ptr(out["fallback"]), _s(stream)),
            "logits_confidence")
    return out


def gather_ln_bf16(src, pairs, div, P, X, stream=None):
    """X[r] = bf16(LN(src[pairs[r] / div])) (src f32): the router's h2 rows in bf16."""
    _count()
    N.check(N.lib.mobile_gather_ln_bf16(N.ptr(src), N.ptr(pairs), int(div), int(P), src.shape[1], N.ptr(X),
                                        _s(stream)), "gather_ln_bf16")
    return X


def gather_bf16(src, pairs, div, P, X, stream=None):
    """X[r] = bf16(src[pairs[r] / div]) (src f32, or bf16 rows: a plain copy)."""
    _count()
    if src.dtype == torch.bfloat16:
        N.check(N.lib.mobile_gather_rows_bf16(N.ptr(src), N.ptr(pairs), int(div), int(P), src.shape[1], N.ptr(X),
                                              _s(stream)), "gather_rows_bf16")
        return X
    N.check(N.lib.mobile_gather_bf16(N.ptr(src), N.ptr(pairs), int(div), int(P), src.shape[1], N.ptr(X), _s(stream)),
            "gather_bf16")
    return X
