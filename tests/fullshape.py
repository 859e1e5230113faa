"""Full-shape parity plumbing (TEST INFRASTRUCTURE): the oracle's KVDecoder
(oracle/moe_ref.py, restating toymoe.py:143-210 / 246-303 with a KV cache)
run on the SAME weights the device holds, read lazily out of the device
layout (weights.py docstring) instead of materialising a 30-60 GB host copy.

Every accessor returns float32 arrays in the reference layout ((in, out)
matrices, toymoe.py:97-126 field shapes): the bf16 device values are exact in
fp32, so the oracle computes in fp32 NumPy/BLAS on bit-identical weights and
the comparison isolates the kernels' arithmetic.  Experts are fetched per
(layer, expert) on demand (a decode step touches only its top-k), with a small
cache; dense per-layer matrices are cached per layer.
"""
from __future__ import annotations

from collections import OrderedDict

import numpy as np
import torch

from oracle import moe_ref as R
from oracle.cpu_baseline import oracle_spec_from


def _np(t: torch.Tensor) -> np.ndarray:
    return t.detach().to(device="cpu", dtype=torch.float32).numpy()


class _PerLayer:
    def __init__(self, fn, n_cache=64):
        self.fn, self.cache, self.n = fn, OrderedDict(), n_cache

    def __getitem__(self, l):
        l = int(l)
        if l not in self.cache:
            if len(self.cache) >= self.n:
                self.cache.popitem(last=False)
            self.cache[l] = self.fn(l)
        return self.cache[l]


class _PerExpert:
    """[layer, e] -> one unpacked matrix of a packed expert (cached by (l, e))."""

    def __init__(self, store, part, d, I, swiglu, cache):
        self.store, self.part, self.d, self.I, self.swiglu, self.cache = store, part, d, I, swiglu, cache

    def _unpack(self, l, e):
        key = (id(self.store), l, e)
        if key not in self.cache.d:
            p = self.store[l, e]
            d, I = self.d, self.I
            r13 = 2 * I if self.swiglu else I
            w13 = _np(p[: r13 * d]).reshape(r13, d)
            w2 = _np(p[r13 * d:]).reshape(d, I)
            if self.swiglu:  # rows interleaved in groups of 8 gate + 8 up (weights.pack_experts)
                g = w13.reshape(I // 8, 2, 8, d)
                gate, up = g[:, 0].reshape(I, d), g[:, 1].reshape(I, d)
            else:
                gate, up = w13, None
            self.cache.put(key, (np.ascontiguousarray(gate.T), None if up is None else np.ascontiguousarray(up.T),
                                 np.ascontiguousarray(w2.T)))
        return self.cache.d[key]

    def __getitem__(self, key):
        l, e = (int(k) for k in key)
        return self._unpack(l, e)[self.part]


class _LRU:
    """Byte-bounded LRU of unpacked experts."""

    def __init__(self, max_bytes):
        self.d, self.max, self.bytes = OrderedDict(), max_bytes, 0

    def put(self, k, v):
        nb = sum(a.nbytes for a in v if a is not None)
        while self.d and self.bytes + nb > self.max:
            _, old = self.d.popitem(last=False)
            self.bytes -= sum(a.nbytes for a in old if a is not None)
        self.d[k] = v
        self.bytes += nb


class _Embed:
    def __init__(self, t: torch.Tensor):
        self.t = t
        self.dtype = np.float32

    def __getitem__(self, idx):
        idx = torch.as_tensor(np.asarray(idx), device=self.t.device, dtype=torch.long)
        return _np(self.t[idx])


def device_oracle(dw) -> R.OracleWeights:
    """OracleWeights view of a DeviceWeights (resident or offloaded experts)."""
    spec = dw.spec
    d, E, I, S, Is = spec.hidden_dim, spec.num_experts, spec.ffn, spec.n_shared, spec.shared_ffn
    sw = spec.activation == "swiglu"
    W = R.OracleWeights.__new__(R.OracleWeights)
    W.spec = oracle_spec_from(spec)
    W.embed = _Embed(dw.embed)
    W.attn_q = _PerLayer(lambda l: np.ascontiguousarray(_np(dw.qkv[l, :d]).T))
    kvd = dw.spec.kv_dim
    W.attn_k = _PerLayer(lambda l: np.ascontiguousarray(_np(dw.qkv[l, d:d + kvd]).T))
    W.attn_v = _PerLayer(lambda l: np.ascontiguousarray(_np(dw.qkv[l, d + kvd:]).T))
    W.attn_o = _PerLayer(lambda l: np.ascontiguousarray(_np(dw.o[l]).T))
    W.router = _PerLayer(lambda l: np.ascontiguousarray(_np(dw.router[l, :E]).T))
    store = dw.experts if dw.experts is not None else dw.host_experts
    cache = _LRU(4 << 30)
    W.expert_in = _PerExpert(store, 0, d, I, sw, cache)
    W.expert_up = _PerExpert(store, 1, d, I, sw, cache) if sw else None
    W.expert_out = _PerExpert(store, 2, d, I, sw, cache)
    W.head = np.ascontiguousarray(_np(dw.head).T)
    W.shared_in = W.shared_up = W.shared_out = W.shared_gate_w = None
    if S:
        scache = _LRU(6 << 30)
        W.shared_in = _PerExpert(dw.shared, 0, d, Is, sw, scache)
        W.shared_up = _PerExpert(dw.shared, 1, d, Is, sw, scache) if sw else None
        W.shared_out = _PerExpert(dw.shared, 2, d, Is, sw, scache)
        if spec.shared_gate == "sigmoid":
            W.shared_gate_w = _PerLayer(lambda l: np.ascontiguousarray(_np(dw.router[l, E:E + S]).T))
    return W


def near_tie(row, a, b, tol) -> bool:
    row = np.asarray(row, dtype=np.float64)
    return abs(row[a] - row[b]) <= tol * max(np.max(np.abs(row)), 1e-30)


def compare_selections(got, want, logits, tol=2e-5):
    """Per-layer selections of one pass: (ok, list of near-tie layers).  A
    layer may differ only where the oracle's own logits make the differing
    positions a near tie (|gap| <= tol * max|logit|)."""
    ties = []
    for l, (g, w) in enumerate(zip(got, want)):
        if list(g) == list(w):
            continue
        row = np.asarray(logits[l], dtype=np.float64)
        scale = max(np.max(np.abs(row)), 1e-30)
        srt = np.sort(row)[::-1]
        k = len(w)
        for a, b in zip(g, w):
            if a != b and abs(row[a] - row[b]) > tol * scale:
                return False, ties
        if set(g) != set(w) and (k >= len(srt) or srt[k - 1] - srt[k] > tol * scale):
            return False, ties
        ties.append(l)
    return True, ties
