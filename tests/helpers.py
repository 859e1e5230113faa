"""Shared test helpers: matched oracle / device weights."""
from __future__ import annotations

import os

import numpy as np

from oracle import moe_ref as R


def ospec(**kw) -> R.OracleSpec:
    return R.OracleSpec(**kw)


def round_bf16(a: np.ndarray) -> np.ndarray:
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).to(torch.float64).numpy()


def matched(spec_kw: dict, dtype: str = "float32", device="cuda"):
    """(OracleWeights, ModelSpec, DeviceModel) on identical weights.

    For bf16 the oracle sees the bf16-rounded values so the comparison isolates
    the kernels' fp32 arithmetic from the storage rounding."""
    from paper_2510_12357_b200 import ModelSpec
    from paper_2510_12357_b200.model import DeviceModel
    from paper_2510_12357_b200.weights import DeviceWeights, HostWeights

    o = R.build_weights(R.OracleSpec(**spec_kw))
    if dtype == "bfloat16":
        for name in ("attn_q", "attn_k", "attn_v", "attn_o", "router", "expert_in", "expert_out", "head",
                     "expert_up", "shared_in", "shared_up", "shared_out", "shared_gate_w"):
            v = getattr(o, name)
            if v is not None:
                setattr(o, name, round_bf16(v))
    ms = ModelSpec(**spec_kw, dtype=dtype)
    hw = HostWeights(o.embed, o.attn_q, o.attn_k, o.attn_v, o.attn_o, o.router, o.expert_in, o.expert_out, o.head,
                     o.expert_up, o.shared_in, o.shared_up, o.shared_out, o.shared_gate_w)
    dm = DeviceModel(DeviceWeights.from_host(ms, hw, device))
    return o, ms, dm


def rel_err(a, b) -> float:
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


# reduced real-shape specs exercising every extension (SwiGLU, shared experts,
# sigmoid shared gate, multi-head attention) at sizes the oracle finishes fast
QWEN_MINI = dict(num_layers=2, num_experts=12, k_big=4, hidden_dim=128, vocab_size=512, seed=5, ffn_dim=64,
                 activation="swiglu", n_shared=1, shared_ffn_dim=256, shared_gate="sigmoid", n_heads=4)
DSEEK_MINI = dict(num_layers=2, num_experts=16, k_big=6, k_little=3, hidden_dim=128, vocab_size=300, seed=6,
                  ffn_dim=64, activation="swiglu", n_shared=2, shared_ffn_dim=64, n_heads=2)
OLMOE_MINI = dict(num_layers=2, num_experts=16, k_big=8, hidden_dim=256, vocab_size=400, seed=8, ffn_dim=128,
                  activation="swiglu", gate_norm="softmax_all", n_heads=4)


NEAR_TIES: list = []  # (test id, layers compared, near-ties) of every selections_agree call
MAX_NEAR_TIES = 2     # near-tie layers tolerated per comparison (reported at the end of the session)


def selections_agree(got, want, logits, tol=2e-5, max_ties=MAX_NEAR_TIES):
    """Layer selections equal, except where the oracle's own logits make the
    order a near-tie (|gap| < tol * max|logit|): then only membership/order
    among near-equal logits may differ, and at most `max_ties` layers may.
    Every call is tallied in NEAR_TIES (printed by tests/conftest.py, never
    silently discarded).  Returns (ok, n_near_ties)."""
    ok, near = _agree(got, want, logits, tol)
    NEAR_TIES.append((os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], len(list(want)), near))
    return ok and near <= max_ties, near


def _agree(got, want, logits, tol):
    near = 0
    for l, (g, w) in enumerate(zip(got, want)):
        if list(g) == list(w):
            continue
        row = np.asarray(logits[l], dtype=np.float64)
        scale = max(np.max(np.abs(row)), 1e-30)
        srt = np.sort(row)[::-1]
        k = len(w)
        # every differing position must be a near tie in the oracle's ranking
        for a, b in zip(g, w):
            if a != b and abs(row[a] - row[b]) > tol * scale:
                return False, near
        if set(g) != set(w) and (k >= len(srt) or srt[k - 1] - srt[k] > tol * scale):
            return False, near
        near += 1
    return True, near

QWEN_MINI_NOPE = dict(QWEN_MINI, embed_scale=1.0, pos_encoding="none", seed=9)
# grouped-query attention (Mixtral-style: 2 key/value heads for 4 query heads), head_dim 32
GQA_MINI = dict(num_layers=2, num_experts=8, k_big=2, k_little=1, hidden_dim=128, vocab_size=320, seed=11, ffn_dim=128,
                activation="swiglu", n_heads=4, n_kv_heads=2, embed_scale=1.0, pos_encoding="none")
