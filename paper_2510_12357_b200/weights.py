"""Weight generation and the HBM layout of the MoBiLE layer.

Host generation follows the reference's seeded draw order exactly for the toy
(toymoe.py:97-126: default_rng(seed), uniform(-1,1)/sqrt(d), embed, q, k, v, o,
router, expert_in, expert_out, head); the real-shape extensions (W3, shared
experts, shared gate) are drawn after that prefix so the toy stream is
unchanged.  Large shapes (d=2048...) are generated directly on the device in
device layout (same distribution, torch RNG) because a host fp64 draw of 14 B
parameters is neither needed nor feasible.

Device layout (all "out-major": rows = output features over the input dim,
row-major), shared by the bulk-copy streaming engine (decode; a 16-row tile
is one contiguous copy whenever the row fits a 4 KB K chunk, else 16 row
copies) and the tcgen05 grouped GEMM (prefill; 2-D/3-D TMA maps over the
same rows).
  router   (L, E + S_gate, d)   rows E.. = Qwen-style sigmoid shared-gate rows
  experts  (L, E, P)            packed per expert: W13 then W2, where
           W13 = (2I, d) SwiGLU gate/up rows interleaved in groups of 8+8
                 (or (I, d) = W_in^T for ReLU), W2 = (d, I) = W_out^T
  shared   (L, S, Ps)           same packing with the shared ffn dim
  qkv      (L, d + 2 kvd, d)    [Wq^T; Wk^T; Wv^T] (one GEMV per layer; kvd = kv_heads x head_dim,
                                = d without grouped-query attention)
  o        (L, d, d)            Wo^T
  head     (V, d)               = head^T
  embed    (V, d) f32
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .spec import ConfigError, ModelSpec

TOY_MAX_HIDDEN, TOY_MAX_VOCAB, TOY_MAX_LAYERS, TOY_MAX_EXPERTS = 512, 4096, 64, 256  # toymoe.py:37-40


def torch_dtype(spec: ModelSpec):
    return torch.bfloat16 if spec.dtype == "bfloat16" else torch.float32


def expert_elems(d: int, I: int, activation: str) -> tuple[int, int]:
    """(elements of W13, elements of the whole packed expert)."""
    r13 = 2 * I if activation == "swiglu" else I
    return r13 * d, r13 * d + d * I


@dataclass
class HostWeights:
    """Reference-layout fp64 weights (the toy's ToyMoE fields + extensions)."""

    embed: np.ndarray
    attn_q: np.ndarray
    attn_k: np.ndarray
    attn_v: np.ndarray
    attn_o: np.ndarray
    router: np.ndarray  # (L, d, E)
    expert_in: np.ndarray  # (L, E, d, I)
    expert_out: np.ndarray  # (L, E, I, d)
    head: np.ndarray  # (d, V)
    expert_up: np.ndarray | None = None
    shared_in: np.ndarray | None = None
    shared_up: np.ndarray | None = None
    shared_out: np.ndarray | None = None
    shared_gate_w: np.ndarray | None = None


def check_toy_limits(spec: ModelSpec) -> None:
    """toymoe.py:100-107 guard rails (the reference-compatible build_model)."""
    for val, lim, name in ((spec.hidden_dim, TOY_MAX_HIDDEN, "hidden_dim"), (spec.vocab_size, TOY_MAX_VOCAB, "vocab_size"),
                           (spec.num_layers, TOY_MAX_LAYERS, "num_layers"), (spec.num_experts, TOY_MAX_EXPERTS, "num_experts")):
        if val > lim:
            raise ConfigError(f"{name} {val} exceeds toy-model limit {lim}")


def init_host_weights(spec: ModelSpec) -> HostWeights:
    rng = np.random.default_rng(spec.seed)
    d, E, L, V, I = spec.hidden_dim, spec.num_experts, spec.num_layers, spec.vocab_size, spec.ffn
    S, Is = spec.n_shared, spec.shared_ffn

    def draw(*shape, fan_in=d):
        return rng.uniform(-1.0, 1.0, size=shape) * (1.0 / np.sqrt(fan_in))

    embed = draw(V, d, fan_in=1.0 / spec.embed_scale**2 if spec.embed_scale else d)
    q, k, v, o = (draw(L, d, d) for _ in range(4))
    router = draw(L, d, E)
    w_in = draw(L, E, d, I)
    w_out = draw(L, E, I, d, fan_in=I)
    head = draw(d, V)
    hw = HostWeights(embed, q, k, v, o, router, w_in, w_out, head)
    if spec.activation == "swiglu":
        hw.expert_up = draw(L, E, d, I)
    if S:
        hw.shared_in = draw(L, S, d, Is)
        if spec.activation == "swiglu":
            hw.shared_up = draw(L, S, d, Is)
        hw.shared_out = draw(L, S, Is, d, fan_in=Is)
        if spec.shared_gate == "sigmoid":
            hw.shared_gate_w = draw(L, d, S)
    return hw


def pack_experts(w_in: torch.Tensor, w_up: torch.Tensor | None, w_out: torch.Tensor) -> torch.Tensor:
    """(..., d, I), (..., d, I), (..., I, d) reference layout -> (..., P) packed device layout."""
    lead = w_in.shape[:-2]
    d, I = w_in.shape[-2], w_in.shape[-1]
    w1t = w_in.transpose(-1, -2)  # (..., I, d)
    if w_up is not None:
        if I % 8:
            raise ConfigError(f"swiglu ffn_dim {I} must be a multiple of 8")
        w3t = w_up.transpose(-1, -2)
        g = torch.stack([w1t.reshape(*lead, I // 8, 8, d), w3t.reshape(*lead, I // 8, 8, d)], dim=-3)
        w13 = g.reshape(*lead, 2 * I, d)
    else:
        w13 = w1t
    w2t = w_out.transpose(-1, -2)  # (..., d, I)
    return torch.cat([w13.contiguous().reshape(*lead, -1), w2t.contiguous().reshape(*lead, -1)], dim=-1).contiguous()


class DeviceWeights:
    """All weights of a model in device layout (experts optionally elsewhere)."""

    def __init__(self, spec: ModelSpec, device, experts_on_device: bool = True):
        self.spec = spec
        self.device = torch.device(device)
        self.wdtype = torch_dtype(spec)
        self.experts_on_device = experts_on_device
        d, I = spec.hidden_dim, spec.ffn
        self.w13_elems, self.expert_elems = expert_elems(d, I, spec.activation)
        self.s_w13_elems, self.shared_elems = expert_elems(d, spec.shared_ffn, spec.activation)
        self.elem_bytes = 2 if self.wdtype == torch.bfloat16 else 4
        self.n_gate_rows = spec.n_shared if spec.shared_gate == "sigmoid" else 0
        self.embed = self.qkv = self.o = None
        self.router = self.experts = self.shared = self.head = None
        self.host_experts = None  # pinned host store when experts are offloaded

    # ---- bytes (for rooflines) ----
    @property
    def expert_bytes(self) -> int:
        return self.expert_elems * self.elem_bytes

    @property
    def shared_bytes(self) -> int:
        return self.shared_elems * self.elem_bytes

    @classmethod
    def from_host(cls, spec: ModelSpec, hw: HostWeights, device, experts_on_device=True) -> "DeviceWeights":
        dw = cls(spec, device, experts_on_device)
        wt, dev = dw.wdtype, dw.device

        def T(a, dtype=wt):
            return torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dtype)

        dw.embed = T(hw.embed, torch.float32)
        tr = lambda a: np.transpose(a, (0, 2, 1))  # noqa: E731  (L, in, out) -> (L, out, in)
        dw.qkv = T(np.concatenate([tr(hw.attn_q), tr(hw.attn_k), tr(hw.attn_v)], axis=1))
        dw.o = T(tr(hw.attn_o))
        rt = np.transpose(hw.router, (0, 2, 1))  # (L, E, d)
        if dw.n_gate_rows:
            rt = np.concatenate([rt, np.transpose(hw.shared_gate_w, (0, 2, 1))], axis=1)
        dw.router = T(rt)
        tt = lambda a: None if a is None else torch.from_numpy(a).to(wt)  # noqa: E731
        packed = pack_experts(tt(hw.expert_in), tt(hw.expert_up), tt(hw.expert_out))
        if experts_on_device:
            dw.experts = packed.to(device=dev, dtype=wt)
        else:
            dw.host_experts = packed.to(dtype=wt).pin_memory()
        if spec.n_shared:
            sp = pack_experts(tt(hw.shared_in), tt(hw.shared_up), tt(hw.shared_out))
            dw.shared = sp.to(device=dev, dtype=wt)
        dw.head = T(np.ascontiguousarray(hw.head.T))
        return dw

    def shard_experts(self, lo: int, hi: int) -> "DeviceWeights":
        """This rank's view for expert parallelism: routed experts [lo, hi),
        everything else (router, shared experts, attention, head) shared."""
        from dataclasses import replace
        sub = DeviceWeights(replace(self.spec, num_experts=hi - lo, k_big=min(self.spec.k_big, hi - lo),
                                    k_little=min(self.spec.k_little, hi - lo)), self.device, True)
        for name in ("embed", "qkv", "o", "router", "shared", "head"):
            setattr(sub, name, getattr(self, name))
        sub.experts = self.experts[:, lo:hi]
        return sub

    def shard_experts_offloaded(self, lo: int, hi: int) -> "DeviceWeights":
        """shard_experts() with the shard's routed experts in pinned host memory
        (contiguous (L, hi - lo, P), the layout OffloadRuntime streams from)."""
        sub = self.shard_experts(lo, hi)
        src = self.experts[:, lo:hi] if self.experts is not None else self.host_experts[:, lo:hi]
        sub.host_experts = src.to("cpu").contiguous().pin_memory()
        sub.experts = None
        sub.experts_on_device = False
        return sub

    def plain(self, w: torch.Tensor) -> torch.Tensor:
        """Row-major (N, K) view of a weight (the device layout is row-major)."""
        return w

    @classmethod
    def random(cls, spec: ModelSpec, device, seed: int = 0, experts_on_device=True) -> "DeviceWeights":
        """Same uniform(-1,1)/sqrt(fan_in) distribution, drawn on the device in device layout."""
        dw = cls(spec, device, experts_on_device)
        dev, wt = dw.device, dw.wdtype
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        d, E, L, V, I, S = spec.hidden_dim, spec.num_experts, spec.num_layers, spec.vocab_size, spec.ffn, spec.n_shared

        def U(*shape, fan_in=d, dtype=wt, device=dev):
            t = torch.empty(*shape, device=dev, dtype=torch.float32)
            t.uniform_(-1.0, 1.0, generator=g).mul_(1.0 / np.sqrt(fan_in))
            return t.to(dtype)

        dw.embed = U(V, d, fan_in=1.0 / spec.embed_scale**2 if spec.embed_scale else d, dtype=torch.float32)
        dw.qkv = U(L, d + 2 * spec.kv_dim, d)
        dw.o = U(L, d, d)
        dw.router = U(L, E + dw.n_gate_rows, d)
        dw.head = U(V, d)
        # packed experts: W13 rows have fan_in d, W2 rows fan_in I
        def experts(n_layer_experts, II, count):
            w13e, tot = expert_elems(d, II, spec.activation)
            t = torch.empty(count, tot, device=dev, dtype=wt)
            a = torch.empty(count, w13e, device=dev, dtype=torch.float32)
            a.uniform_(-1.0, 1.0, generator=g).mul_(1.0 / np.sqrt(d))
            t[:, :w13e] = a.to(wt)
            del a
            b = torch.empty(count, tot - w13e, device=dev, dtype=torch.float32)
            b.uniform_(-1.0, 1.0, generator=g).mul_(1.0 / np.sqrt(II))
            t[:, w13e:] = b.to(wt)
            return t

        if experts_on_device:
            dw.experts = torch.empty(L, E, dw.expert_elems, device=dev, dtype=wt)
            for l in range(L):
                dw.experts[l] = experts(E, I, E)
        else:
            dw.host_experts = torch.empty(L, E, dw.expert_elems, dtype=wt, pin_memory=True)
            for l in range(L):
                dw.host_experts[l].copy_(experts(E, I, E))
        if S:
            dw.shared = torch.empty(L, S, dw.shared_elems, device=dev, dtype=wt)
            for l in range(L):
                dw.shared[l] = experts(S, spec.shared_ffn, S)
        torch.cuda.synchronize(dev)
        return dw

    def device_bytes(self) -> int:
        n = 0
        for t in (self.embed, self.qkv, self.o, self.router, self.experts, self.shared, self.head):
            if t is not None:
                n += t.numel() * t.element_size()
        return n
