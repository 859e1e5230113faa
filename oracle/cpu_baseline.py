"""CPU reference leg of bench.py -- TEST/BENCH INFRASTRUCTURE ONLY.

Times the oracle's NumPy restatement of the KV-cached MoBiLE decode
(moe_ref.KVDecoder + Algorithm 1) at a real model shape in fp32 on the host
cores.  The reference package itself cannot build d=2048 models
(toymoe.py:100-107), so this port is the CPU path (`kind: "port"`).

Memory bound: a full fp32 Qwen1.5-MoE copy is 57 GB, so the per-layer
matrices are drawn into small pools and layers/experts alias pool entries.
Every pool is far larger than the host LLC, so each token still streams the
same number of distinct-from-cache bytes as the full model would; the
aliasing only bounds RAM and generation time.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import moe_ref as R


class _ByLayer:
    def __init__(self, pool):
        self.pool = pool

    def __getitem__(self, key):
        if isinstance(key, tuple):
            return self.pool[key[0] % len(self.pool)][key[1:]]
        return self.pool[key % len(self.pool)]


class _ByExpert:
    def __init__(self, pool, E):
        self.pool, self.E = pool, E

    def __getitem__(self, key):
        l, e = key
        return self.pool[(l * self.E + e) % len(self.pool)]


def aliased_weights(spec: R.OracleSpec, layer_pool=4, expert_pool=64, seed=0) -> R.OracleWeights:
    rng = np.random.default_rng(seed)
    d, E, L, V, I, S, Is = (spec.hidden_dim, spec.num_experts, spec.num_layers, spec.vocab_size, spec.ffn_dim,
                            spec.n_shared, spec.shared_ffn_dim)

    def U(*shape, fan_in=d):
        return (rng.random(shape, dtype=np.float32) * 2 - 1) * np.float32(1 / np.sqrt(fan_in))

    lp = min(layer_pool, L)
    ep = min(expert_pool, L * E)
    kvd = spec.kv_dim
    attn = [_ByLayer([U(d, w) for _ in range(lp)]) for w in (d, kvd, kvd, d)]
    w_in = _ByExpert([U(d, I) for _ in range(ep)], E)
    w_up = _ByExpert([U(d, I) for _ in range(ep)], E) if spec.activation == "swiglu" else None
    w_out = _ByExpert([U(I, d, fan_in=I) for _ in range(ep)], E)
    W = R.OracleWeights(spec, U(V, d, fan_in=1.0 / spec.embed_scale**2 if spec.embed_scale else d), attn[0], attn[1], attn[2], attn[3], U(L, d, E), w_in, w_out, U(d, V), w_up)
    if S:
        W.shared_in = _ByLayer([U(S, d, Is) for _ in range(lp)])
        W.shared_up = _ByLayer([U(S, d, Is) for _ in range(lp)]) if spec.activation == "swiglu" else None
        W.shared_out = _ByLayer([U(S, Is, d, fan_in=Is) for _ in range(lp)])
        if spec.shared_gate == "sigmoid":
            W.shared_gate_w = U(L, d, S)
    return W


def oracle_spec_from(ms) -> R.OracleSpec:
    return R.OracleSpec(num_layers=ms.num_layers, num_experts=ms.num_experts, k_big=ms.k_big, k_little=ms.k_little,
                        hidden_dim=ms.hidden_dim, vocab_size=ms.vocab_size, eos_token=ms.eos_token, seed=ms.seed,
                        ffn_dim=ms.ffn, activation=ms.activation, n_shared=ms.n_shared,
                        shared_ffn_dim=ms.shared_ffn, shared_gate=ms.shared_gate, gate_norm=ms.gate_norm,
                        n_heads=ms.n_heads, n_kv_heads=ms.kv_heads, logit_scale=ms.logit_scale,
                        embed_scale=ms.embed_scale,
                        pos_encoding=ms.pos_encoding)


# The bench workload's shape (BASELINE.json configs[2], C3) restated on the
# oracle side, so bench.py's CPU legs never import the product package:
# Qwen1.5-MoE-A2.7B (d2048, 24 layers, 60 routed experts top-4 / little top-2,
# one 5632-wide sigmoid-gated shared expert, V151936), unit-scale embeddings,
# no additive position code (paper_2510_12357_b200/presets.py QWEN15_MOE).
C3_SPEC = R.OracleSpec(num_layers=24, num_experts=60, k_big=4, k_little=2, hidden_dim=2048, vocab_size=151936,
                       ffn_dim=1408, activation="swiglu", n_shared=1, shared_ffn_dim=5632, shared_gate="sigmoid",
                       n_heads=16, embed_scale=1.0, pos_encoding="none")


# The other BASELINE.json configs on the oracle side (presets.py OLMOE /
# DEEPSEEK_MOE_16B / MIXTRAL_8X7B), for bench.py's per-config CPU legs.
C2_SPEC = R.OracleSpec(num_layers=16, num_experts=64, k_big=8, k_little=4, hidden_dim=2048, vocab_size=50304,
                       ffn_dim=1024, activation="swiglu", n_heads=16, embed_scale=1.0, pos_encoding="none")
C4_SPEC = R.OracleSpec(num_layers=27, num_experts=64, k_big=6, k_little=3, hidden_dim=2048, vocab_size=102400,
                       ffn_dim=1408, activation="swiglu", n_shared=2, shared_ffn_dim=1408, n_heads=16,
                       embed_scale=1.0, pos_encoding="none")
C5_SPEC = R.OracleSpec(num_layers=32, num_experts=8, k_big=2, k_little=1, hidden_dim=4096, vocab_size=32000,
                       ffn_dim=14336, activation="swiglu", n_heads=32, n_kv_heads=8, embed_scale=1.0,
                       pos_encoding="none")
SPECS = {"c2": C2_SPEC, "c3": C3_SPEC, "c4": C4_SPEC, "c5": C5_SPEC}


def c3_slots(cap_bytes: int, reserved_bytes: int, spec: R.OracleSpec = C3_SPEC) -> int:
    """hbm_expert_slots (config.py:204-218) on the bf16 device sizes of `spec`
    (expert = 3 d I, dense/layer = qkv+o + router + shared + shared gate)."""
    d, per = spec.hidden_dim, 2
    expert = 3 * d * spec.ffn_dim * per
    dense = (2 * d * d + 2 * d * spec.kv_dim) * per + d * spec.num_experts * per + spec.n_shared * 3 * d * spec.shared_ffn_dim * per \
        + (spec.n_shared * d * per if spec.shared_gate == "sigmoid" else 0)
    return R.hbm_expert_slots(spec.num_layers, dense, cap_bytes, reserved_bytes, expert, spec.k_big)


def synthetic_context(dec: R.KVDecoder, n: int, seed: int = 3) -> None:
    """Fill the KV cache with `n` random positions (a bounded stand-in for
    prefilling an n-token prompt: decode cost depends on the cache length,
    not its contents)."""
    rng = np.random.default_rng(seed)
    d = dec.W.spec.kv_dim
    for l in range(dec.W.spec.num_layers):
        dec.k_cache[l] = rng.standard_normal((n, d), dtype=np.float32)
        dec.v_cache[l] = rng.standard_normal((n, d), dtype=np.float32)


def time_decode(W: R.OracleWeights, prompt, flags, warmup: int, steps: int, gamma=0.7, context: int = 0):
    """MoBiLE KV decode on the CPU: returns (seconds for `steps` tokens,
    fallbacks).  `context` > 0: start from a synthetic cache of that many
    positions instead of prefilling prompt[:-1]."""
    s = W.spec
    dec = R.KVDecoder(W)
    if context:
        synthetic_context(dec, context)
    else:
        dec.prefill(list(prompt[:-1]))
    last = prompt[-1]
    fallbacks = 0
    t0 = None
    for i in range(warmup + steps):
        if i == warmup:
            t0 = time.perf_counter()
        probs, states, _, kv = dec.run([last], s.k_little)
        fb = bool(flags[i]) if flags is not None else R.should_fallback(probs, gamma)
        if fb:
            probs, _, _, kv = dec.run([last], s.k_big, states)
            if i >= warmup:
                fallbacks += 1
        dec.commit(kv)
        last = int(np.argmax(probs))
    return time.perf_counter() - t0, fallbacks


def cores() -> int:
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
