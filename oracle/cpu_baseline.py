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
    attn = [_ByLayer([U(d, d) for _ in range(lp)]) for _ in range(4)]
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
                        n_heads=ms.n_heads, logit_scale=ms.logit_scale, embed_scale=ms.embed_scale,
                        pos_encoding=ms.pos_encoding)


def time_decode(W: R.OracleWeights, prompt, flags, warmup: int, steps: int, gamma=0.7):
    """MoBiLE KV decode on the CPU: returns (seconds for `steps` tokens, fallbacks)."""
    s = W.spec
    dec = R.KVDecoder(W)
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
