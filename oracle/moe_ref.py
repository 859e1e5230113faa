"""NumPy restatement of the reference MoBiLE path -- TEST INFRASTRUCTURE ONLY.

See `oracle/__init__.py` for the import rule.  Every function cites the
reference line it restates (paths relative to `/root/reference/pkg/src/moesim/`).

Toy settings (activation="relu", ffn_dim == hidden_dim, no shared experts,
selected-softmax gating, one attention head) reproduce `toymoe.forward` /
`generate` bit-for-bit in fp64: the arithmetic expressions below are the
reference's own, in the same order.  Everything else (SwiGLU, shared experts,
sigmoid shared gate, HF "softmax over all" gating, multi-head attention,
KV-cache decode) is an extension the reference does not pin -- parity for it
is against this restatement only.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

LOGIT_SCALE = 24.0  # toymoe.py:34
LN_EPS = 1e-5  # toymoe.py:36

ACCEPTED_LITTLE = "Little"  # toymoe.py:28
ACCEPTED_BIG = "BigFallback"  # toymoe.py:29


# ---------------------------------------------------------------------------
# spec


@dataclass(frozen=True)
class OracleSpec:
    """ModelSpec (config.py:75-115) plus the real-shape extensions."""

    num_layers: int
    num_experts: int
    k_big: int
    k_little: int = 0  # 0 -> max(1, k_big // 2)  (config.py:90-92)
    hidden_dim: int = 64
    vocab_size: int = 256
    eos_token: int = 0
    seed: int = 0
    ffn_dim: int = 0  # 0 -> hidden_dim (the toy expert is d -> d -> d)
    activation: str = "relu"  # "relu" (toy) | "swiglu"
    n_shared: int = 0
    shared_ffn_dim: int = 0  # 0 -> ffn_dim
    shared_gate: str = "none"  # "none" | "sigmoid" (Qwen-style)
    gate_norm: str = "selected_softmax"  # toymoe.py:201 | "softmax_all" (HF norm_topk_prob=False)
    n_heads: int = 1
    n_kv_heads: int = 0  # 0 -> n_heads (extension: grouped-query attention)
    logit_scale: float = LOGIT_SCALE
    embed_scale: float = 0.0  # 0 -> 1/sqrt(d) as the toy (toymoe.py:109-112)
    pos_encoding: str = "sinusoidal"  # toymoe.py:135-140 | "none" (extension)

    def __post_init__(self):
        if self.k_little == 0:
            object.__setattr__(self, "k_little", max(1, self.k_big // 2))
        if self.ffn_dim == 0:
            object.__setattr__(self, "ffn_dim", self.hidden_dim)
        if self.shared_ffn_dim == 0:
            object.__setattr__(self, "shared_ffn_dim", self.ffn_dim)
        if self.n_kv_heads == 0:
            object.__setattr__(self, "n_kv_heads", self.n_heads)

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * (self.hidden_dim // self.n_heads)


# ---------------------------------------------------------------------------
# elementary ops


def top_k(logits, k: int) -> list[int]:
    """toymoe.py:80-88: descending, ties to the lower index (stable argsort)."""
    logits = np.asarray(logits)
    if k > logits.shape[-1]:
        raise ValueError(f"k ({k}) exceeds number of experts ({logits.shape[-1]})")
    if not np.all(np.isfinite(logits)):
        raise ValueError("router logits must be finite")
    order = np.argsort(-logits, kind="stable")
    return [int(i) for i in order[:k]]


def reference_top_k(logits, k: int) -> list[int]:
    """Independent pure-Python ordering (test_toymoe.py:26-28 style)."""
    return sorted(range(len(logits)), key=lambda i: (-logits[i], i))[:k]


def softmax(x: np.ndarray) -> np.ndarray:
    """toymoe.py:91-94."""
    x = x - np.max(x)
    e = np.exp(x)
    return e / e.sum()


def layer_norm(x: np.ndarray) -> np.ndarray:
    """toymoe.py:129-132: no affine, population variance, eps 1e-5."""
    mean = x.mean(axis=-1, keepdims=True)
    var = x.var(axis=-1, keepdims=True)
    return (x - mean) / np.sqrt(var + LN_EPS)


def positional(n: int, d: int, start: int = 0) -> np.ndarray:
    """toymoe.py:135-140 (rows start..start+n-1)."""
    pos = np.arange(start, start + n)[:, None]
    dim = np.arange(d)[None, :]
    angle = pos / np.power(10000.0, (2 * (dim // 2)) / d)
    return np.where(dim % 2 == 0, np.sin(angle), np.cos(angle))


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


def sigmoid(x: np.ndarray) -> np.ndarray:
    return 1.0 / (1.0 + np.exp(-x))


# ---------------------------------------------------------------------------
# weights


@dataclass
class OracleWeights:
    spec: OracleSpec
    embed: np.ndarray  # (V, d)
    attn_q: np.ndarray  # (L, d, d)
    attn_k: np.ndarray
    attn_v: np.ndarray
    attn_o: np.ndarray
    router: np.ndarray  # (L, d, E)
    expert_in: np.ndarray  # (L, E, d, I)   (W1 / gate for swiglu)
    expert_out: np.ndarray  # (L, E, I, d)  (W2)
    head: np.ndarray  # (d, V)
    expert_up: np.ndarray | None = None  # (L, E, d, I) W3, swiglu only
    shared_in: np.ndarray | None = None  # (L, S, d, Is)
    shared_up: np.ndarray | None = None  # (L, S, d, Is)
    shared_out: np.ndarray | None = None  # (L, S, Is, d)
    shared_gate_w: np.ndarray | None = None  # (L, d, S) sigmoid gate

    def astype(self, dtype) -> "OracleWeights":
        out = {}
        for k, v in self.__dict__.items():
            out[k] = v.astype(dtype) if isinstance(v, np.ndarray) else v
        return OracleWeights(**out)


def build_weights(spec: OracleSpec) -> OracleWeights:
    """toymoe.py:97-126: default_rng(seed), uniform(-1, 1) * scale, fixed draw order.

    The toy draws embed, q, k, v, o, router, expert_in, expert_out, head with
    scale 1/sqrt(d).  Extensions draw after that prefix so the toy stream is
    unchanged: expert_up (swiglu) is drawn after expert_out/head, then the
    shared-expert tensors, each scaled 1/sqrt(fan_in).  (The toy's guard rails
    on d/V, toymoe.py:100-107, are not applied here: the oracle also builds
    reduced real-shape layers.)
    """
    rng = np.random.default_rng(spec.seed)
    d, E, L, V = spec.hidden_dim, spec.num_experts, spec.num_layers, spec.vocab_size
    I, S, Is = spec.ffn_dim, spec.n_shared, spec.shared_ffn_dim

    def mat(*shape, fan_in=d):
        return rng.uniform(-1.0, 1.0, size=shape) * (1.0 / np.sqrt(fan_in))

    embed = mat(V, d, fan_in=1.0 / spec.embed_scale**2 if spec.embed_scale else d)
    kvd = spec.kv_dim  # = d unless grouped-query attention
    q, k, v, o = mat(L, d, d), mat(L, d, kvd), mat(L, d, kvd), mat(L, d, d)
    router = mat(L, d, E)
    w_in = mat(L, E, d, I)
    w_out = mat(L, E, I, d, fan_in=I)
    head = mat(d, V)
    w_up = mat(L, E, d, I) if spec.activation == "swiglu" else None
    s_in = s_up = s_out = s_g = None
    if S > 0:
        s_in = mat(L, S, d, Is)
        s_up = mat(L, S, d, Is) if spec.activation == "swiglu" else None
        s_out = mat(L, S, Is, d, fan_in=Is)
        if spec.shared_gate == "sigmoid":
            s_g = mat(L, d, S)
    return OracleWeights(spec, embed, q, k, v, o, router, w_in, w_out, head,
                         w_up, s_in, s_up, s_out, s_g)


# ---------------------------------------------------------------------------
# the MoE block (toymoe.py:188-207), carved out with per-token width/replay


def _expert(h, w_in, w_up, w_out, activation):
    """toymoe.py:203-204 (relu) / SwiGLU extension."""
    if activation == "relu":
        hidden = np.maximum(h @ w_in, 0.0)
    else:
        hidden = silu(h @ w_in) * (h @ w_up)
    return hidden @ w_out


@dataclass
class MoEOut:
    out: np.ndarray  # (T, d) moe contribution (residual NOT added)
    logits: np.ndarray  # (T, E) own router logits
    selections: list[list[int]]  # per token
    gates: list[np.ndarray]  # per token, selection order


def route_token(own_logits, k, replay_row=None, reuse_gates=False, gate_norm="selected_softmax"):
    """Selection + gates for one token (toymoe.py:194-201)."""
    if replay_row is not None:
        sel = top_k(replay_row, k)
        gate_logits = replay_row if reuse_gates else own_logits
    else:
        sel = top_k(own_logits, k)
        gate_logits = own_logits
    if gate_norm == "selected_softmax":
        gates = softmax(gate_logits[sel])
    else:  # HF norm_topk_prob=False: softmax over all experts, no renormalisation
        gates = softmax(gate_logits)[sel]
    return sel, gates


def moe_block(W: OracleWeights, layer: int, h2: np.ndarray, k_tok, replay_rows=None,
              replay_mask=None, reuse_gates=False) -> MoEOut:
    """toymoe.py:188-207 for T tokens; token t uses width k_tok[t] and, if
    replay_mask[t], selects top_k(replay_rows[t]) (toymoe.py:195-198)."""
    spec = W.spec
    logits = h2 @ W.router[layer]  # toymoe.py:189 (one GEMM over all rows)
    moe_out = np.zeros_like(h2)
    sels, gates_all = [], []
    for pos in range(h2.shape[0]):
        rep = None
        if replay_mask is not None and replay_mask[pos]:
            rep = replay_rows[pos]
        sel, gates = route_token(logits[pos], int(k_tok[pos]), rep, reuse_gates, spec.gate_norm)
        for g, e in zip(gates, sel):
            w_up = W.expert_up[layer, e] if W.expert_up is not None else None
            moe_out[pos] += g * _expert(h2[pos], W.expert_in[layer, e], w_up,
                                        W.expert_out[layer, e], spec.activation)
        sels.append(sel)
        gates_all.append(gates)
    if spec.n_shared:
        for s in range(spec.n_shared):
            w_up = W.shared_up[layer, s] if W.shared_up is not None else None
            y = _expert(h2, W.shared_in[layer, s], w_up, W.shared_out[layer, s], spec.activation)
            if spec.shared_gate == "sigmoid":
                y = sigmoid(h2 @ W.shared_gate_w[layer][:, s:s + 1]) * y
            moe_out += y
    return MoEOut(moe_out, logits, sels, gates_all)


def attention(W: OracleWeights, layer: int, h: np.ndarray, k_cache=None, v_cache=None):
    """toymoe.py:178-186, generalised to n_heads (one head = the reference).

    With caches, `h` holds only the new rows and attends to cache + itself
    (causal).  Returns (attn_out @ Wo, key rows, value rows).
    """
    spec = W.spec
    d = spec.hidden_dim
    q = h @ W.attn_q[layer]
    key = h @ W.attn_k[layer]
    v = h @ W.attn_v[layer]
    if k_cache is not None and len(k_cache):
        kk = np.concatenate([k_cache, key], axis=0)
        vv = np.concatenate([v_cache, v], axis=0)
    else:
        kk, vv = key, v
    n_new, n_all = q.shape[0], kk.shape[0]
    offset = n_all - n_new
    mask = np.triu(np.full((n_new, n_all), -np.inf), k=1 + offset)
    H = spec.n_heads
    if H == 1:
        scores = q @ kk.T / np.sqrt(d) + mask
        scores -= scores.max(axis=-1, keepdims=True)
        attn = np.exp(scores)
        attn /= attn.sum(axis=-1, keepdims=True)
        out = attn @ vv
    else:
        hd = d // H
        grp = H // spec.n_kv_heads  # query heads per key/value head (1 = multi-head)
        out = np.empty_like(q)
        for hh in range(H):
            sl = slice(hh * hd, (hh + 1) * hd)
            kv = slice((hh // grp) * hd, (hh // grp + 1) * hd)
            scores = q[:, sl] @ kk[:, kv].T / np.sqrt(hd) + mask
            scores -= scores.max(axis=-1, keepdims=True)
            attn = np.exp(scores)
            attn /= attn.sum(axis=-1, keepdims=True)
            out[:, sl] = attn @ vv[:, kv]
    return out @ W.attn_o[layer], key, v


def head_probs(W: OracleWeights, x_last: np.ndarray) -> np.ndarray:
    """toymoe.py:209-210: softmax(LN(x_last) @ head * 24)."""
    out = layer_norm(x_last) @ W.head * W.spec.logit_scale
    return softmax(out)


# ---------------------------------------------------------------------------
# recompute forward + generate (the reference's functional semantics)


@dataclass
class ForwardOut:
    probs: np.ndarray
    router_states: np.ndarray
    selections: list[list[int]]


def forward(W: OracleWeights, tokens, k: int, replay_states=None, reuse_gates=False) -> ForwardOut:
    """toymoe.py:143-210 (full-sequence recompute; replay at the final position)."""
    spec = W.spec
    if not tokens:
        raise ValueError("token sequence is empty")
    for t in tokens:
        if not (0 <= t < spec.vocab_size):
            raise ValueError(f"token {t} outside vocab [0, {spec.vocab_size})")
    if replay_states is not None:
        replay_states = np.asarray(replay_states, dtype=float)
        if replay_states.shape != (spec.num_layers, spec.num_experts):
            raise ValueError(f"router states shape {replay_states.shape} does not match "
                             f"(num_layers, num_experts) = ({spec.num_layers}, {spec.num_experts})")
    n, d = len(tokens), spec.hidden_dim
    x = W.embed[np.asarray(tokens)] + positional(n, d)
    states = np.empty((spec.num_layers, spec.num_experts))
    selections = []
    k_tok = np.full(n, k)
    mask = None
    if replay_states is not None:
        mask = np.zeros(n, dtype=bool)
        mask[-1] = True
    for layer in range(spec.num_layers):
        h = layer_norm(x)
        a, _, _ = attention(W, layer, h)
        x = x + a
        h2 = layer_norm(x)
        rep_rows = None
        if replay_states is not None:
            rep_rows = np.zeros((n, spec.num_experts))
            rep_rows[-1] = replay_states[layer]
        mo = moe_block(W, layer, h2, k_tok, rep_rows, mask, reuse_gates)
        states[layer] = mo.logits[-1]
        selections.append(mo.selections[-1])
        x = x + mo.out
    return ForwardOut(head_probs(W, x[-1]), states, selections)


@dataclass
class Decision:
    token: int
    accepted_by: str
    confidence: float
    little_selections: list
    big_selections: list | None = None
    router_states: np.ndarray | None = None


def _sample(probs, sampling, temperature, rng) -> int:
    """toymoe.py:239-243."""
    if sampling == "Temperature":
        logp = np.log(probs) / temperature
        return int(rng.choice(len(probs), p=softmax(logp)))
    return int(np.argmax(probs))


def generate(W: OracleWeights, prompt, gamma: float, max_len: int, sampling="Greedy",
             temperature=1.0, sampling_seed=0, reuse_gates=False, record_router_states=False):
    """toymoe.py:246-303 (Algorithm 1, recompute semantics)."""
    if not prompt:
        raise ValueError("prompt is empty")
    if max_len < 1:
        raise ValueError(f"max_len must be >= 1, got {max_len}")
    spec = W.spec
    rng = np.random.default_rng(sampling_seed)
    tokens = list(prompt)
    decisions = []
    while len(decisions) < max_len:
        little = forward(W, tokens, spec.k_little)
        confidence = float(little.probs.max())
        if should_fallback(little.probs, gamma):
            big = forward(W, tokens, spec.k_big, little.router_states, reuse_gates)
            token = _sample(big.probs, sampling, temperature, rng)
            decisions.append(Decision(token, ACCEPTED_BIG, confidence, little.selections,
                                      big.selections, little.router_states))
        else:
            token = _sample(little.probs, sampling, temperature, rng)
            decisions.append(Decision(token, ACCEPTED_LITTLE, confidence, little.selections,
                                      None, little.router_states if record_router_states else None))
        tokens.append(token)
        if token == spec.eos_token:
            break
    return tokens, decisions


# ---------------------------------------------------------------------------
# KV-cache decode (extension; the build's perf-path semantics)


class KVDecoder:
    """One sequence, KV-cached.  A position's K/V rows come from the pass whose
    output was accepted (the big pass overwrites on fallback).  The prompt's
    context positions [0, n-1) are prefilled at width `prefill_k` (k_big by
    default); every decision is one decode step at one position."""

    def __init__(self, W: OracleWeights, prefill_k: int | None = None):
        self.W = W
        s = W.spec
        self.prefill_k = s.k_big if prefill_k is None else prefill_k
        dt = W.embed.dtype
        self.k_cache = [np.zeros((0, s.kv_dim), dtype=dt) for _ in range(s.num_layers)]
        self.v_cache = [np.zeros((0, s.kv_dim), dtype=dt) for _ in range(s.num_layers)]

    @property
    def length(self) -> int:
        return self.k_cache[0].shape[0]

    def run(self, tokens, k, replay_states=None, reuse_gates=False):
        """Process `tokens` at positions length.., return (probs_last, states_last,
        selections_last, new_kv).  Does NOT commit the K/V rows."""
        W, s = self.W, self.W.spec
        n = len(tokens)
        pe = positional(n, s.hidden_dim, self.length) if s.pos_encoding != "none" else np.zeros((n, s.hidden_dim))
        x = W.embed[np.asarray(tokens)] + pe.astype(W.embed.dtype)
        states = np.empty((s.num_layers, s.num_experts))
        sels, new_kv = [], []
        mask = None
        if replay_states is not None:
            mask = np.zeros(n, dtype=bool)
            mask[-1] = True
        for layer in range(s.num_layers):
            h = layer_norm(x)
            a, key, v = attention(W, layer, h, self.k_cache[layer], self.v_cache[layer])
            new_kv.append((key, v))
            x = x + a
            h2 = layer_norm(x)
            rep = None
            if replay_states is not None:
                rep = np.zeros((n, s.num_experts))
                rep[-1] = replay_states[layer]
            mo = moe_block(W, layer, h2, np.full(n, k), rep, mask, reuse_gates)
            states[layer] = mo.logits[-1]
            sels.append(mo.selections[-1])
            x = x + mo.out
        return head_probs(W, x[-1]), states, sels, new_kv

    def commit(self, new_kv):
        for layer, (key, v) in enumerate(new_kv):
            self.k_cache[layer] = np.concatenate([self.k_cache[layer], key], axis=0)
            self.v_cache[layer] = np.concatenate([self.v_cache[layer], v], axis=0)

    def prefill(self, tokens):
        if tokens:
            _, _, _, kv = self.run(tokens, self.prefill_k)
            self.commit(kv)


def generate_kv(W: OracleWeights, prompt, gamma: float, max_len: int, reuse_gates=False,
                prefill_k=None, fallback_flags=None):
    """Algorithm 1 over a KV cache (greedy).  `fallback_flags` (per decision)
    overrides the confidence rule, like engine.injected_fallback_flags."""
    if not prompt:
        raise ValueError("prompt is empty")
    s = W.spec
    dec = KVDecoder(W, prefill_k)
    dec.prefill(list(prompt[:-1]))
    tokens = list(prompt)
    decisions = []
    while len(decisions) < max_len:
        last = tokens[-1]
        probs, states, lsel, kv = dec.run([last], s.k_little)
        confidence = float(probs.max())
        fb = should_fallback(probs, gamma)
        if fallback_flags is not None:
            fb = bool(fallback_flags[len(decisions)])
        if fb:
            bprobs, _, bsel, bkv = dec.run([last], s.k_big, states, reuse_gates)
            dec.commit(bkv)
            token = int(np.argmax(bprobs))
            decisions.append(Decision(token, ACCEPTED_BIG, confidence, lsel, bsel, states))
        else:
            dec.commit(kv)
            token = int(np.argmax(probs))
            decisions.append(Decision(token, ACCEPTED_LITTLE, confidence, lsel, None, None))
        tokens.append(token)
        if token == s.eos_token:
            break
    return tokens, decisions


# ---------------------------------------------------------------------------
# policy (policy.py)


def should_fallback(probs, gamma: float) -> bool:
    """policy.py:69-79: strict `>` accepts; |sum-1| > 1e-4 is an error."""
    probs = np.asarray(probs, dtype=float)
    total = float(probs.sum())
    if abs(total - 1.0) > 1e-4:
        raise ValueError(f"probability vector sums to {total}, expected 1 within 1e-4")
    return float(probs.max()) <= gamma


def build_mobile_plan(router_states, k_big: int, lookahead: int):
    """policy.py:86-106. Returns (targets [[(l,e)]], entries [(issue, l, e, after_routing)])."""
    if lookahead < 1:
        raise ValueError(f"lookahead must be >= 1, got {lookahead}")
    states = np.asarray(router_states, dtype=float)
    if states.ndim != 2:
        raise ValueError(f"router states must be 2-D (layers x experts), got shape {states.shape}")
    targets, entries = [], []
    for layer in range(states.shape[0]):
        chosen = [(layer, e) for e in top_k(states[layer], k_big)]
        targets.append(chosen)
        issue = max(0, layer - lookahead)
        entries.extend((issue, l, e, False) for (l, e) in chosen)
    entries.sort(key=lambda t: (t[0], t[1], t[2]))
    return targets, entries


def on_demand_selection(selection):
    """policy.py:109-116."""
    entries = []
    for layer, chosen in enumerate(selection):
        if not chosen:
            raise ValueError(f"layer {layer} has an empty expert selection")
        entries.extend((l, l, e, True) for (l, e) in chosen)
    entries.sort(key=lambda t: (t[0], t[1], t[2]))
    return [list(s) for s in selection], entries


def injected_fallback_flags(n_tokens: int, ratio: float) -> list[bool]:
    """engine.py:271-277."""
    if not (0.0 <= ratio <= 1.0):
        raise ValueError(f"fallback ratio outside [0, 1]: {ratio}")
    return [int((i + 1) * ratio + 1e-9) > int(i * ratio + 1e-9) for i in range(n_tokens)]


def hbm_expert_slots(num_layers, dense_bytes_per_layer, hbm_capacity, reserved, expert_bytes, k_big):
    """config.py:204-218."""
    budget = hbm_capacity - num_layers * dense_bytes_per_layer - reserved
    slots = budget // expert_bytes
    if slots < k_big:
        raise ValueError(f"hbm_capacity {hbm_capacity} leaves room for {slots} expert slots; "
                         f"need at least k_big={k_big}")
    return int(slots)


# ---------------------------------------------------------------------------
# memory (memory.py)


class CapacityDeadlockRef(RuntimeError):
    pass


@dataclass
class ChannelRef:
    """memory.py:29-44."""

    t_xfer: float
    busy_until: float = 0.0
    transfers_issued: int = 0

    def issue(self, now: float) -> float:
        start = max(now, self.busy_until)
        self.busy_until = start + self.t_xfer
        self.transfers_issued += 1
        return self.busy_until


@dataclass
class CacheRef:
    """memory.py:65-181 restated with a dict (insertion order = LRU order)."""

    slots: int
    ready: dict = field(default_factory=dict)
    pins: set = field(default_factory=set)
    hits: int = 0
    coalesced: int = 0
    issued: int = 0
    evictions: int = 0
    deferrals: int = 0

    def request(self, key, now, channel, speculative=False):
        if key in self.ready:
            r = self.ready.pop(key)
            self.ready[key] = r  # move to MRU
            if r <= now:
                self.hits += 1
                return ("hit", r)
            self.coalesced += 1
            return ("in_flight", r)
        if len(self.ready) >= self.slots and not self._evict_one(now):
            if speculative:
                self.deferrals += 1
                return None
            raise CapacityDeadlockRef(f"no evictable slot for {key}")
        r = channel.issue(now)
        self.ready[key] = r
        self.issued += 1
        return ("issued", r)

    def _evict_one(self, now):
        for key, r in self.ready.items():
            if key in self.pins or r > now:
                continue
            del self.ready[key]
            self.evictions += 1
            return True
        return False

    def evict_lru(self, n, now=None):
        if now is None:
            now = float("inf")
        victims = [k for k, r in self.ready.items() if k not in self.pins and r <= now][:n]
        if len(victims) < n:
            raise ValueError(f"asked to evict {n} experts but only {len(victims)} are unpinned")
        for k in victims:
            del self.ready[k]
            self.evictions += 1
        return victims

    def pin(self, key):
        self.pins.add(key)

    def unpin(self, key):
        self.pins.discard(key)

    def token_end(self):
        self.pins.clear()
