"""Model shapes of the BASELINE.json configs (C1-C5).

Real shapes come from the public model configs; the reference
itself only builds the toy C1.  Deviations from the original models, kept so
the MoBiLE layer semantics stay the reference's: LayerNorm without affine,
no rotary positions, grouped-query attention where the model has it (Mixtral:
8 key/value heads for 32 query heads), selected-softmax gating (toymoe.py:201; the HF models
use softmax-over-all, available as gate_norm="softmax_all"), DeepSeek's one
dense first layer omitted (27 MoE layers).

Random-init embeddings are drawn at unit scale (embed_scale=1.0, i.e.
uniform(-1, 1)) and no additive position code is used for the real shapes
(the modelled models use rotary positions, which never enter the residual
stream): with the toy's 1/sqrt(d) embeddings plus additive sinusoids, the
position code dominates LN(x) at d=2048, consecutive decode tokens route to
nearly the same experts and the expert cache almost never misses -- unlike
trained models, whose residual stream is token-dominated.  The toy keeps the
reference's choices.
"""

from __future__ import annotations

from dataclasses import replace

from .spec import HardwareSpec, ModelSpec

C1_TINY = ModelSpec(num_layers=2, num_experts=16, k_big=4, k_little=2, hidden_dim=256, vocab_size=256, seed=0)

OLMOE = ModelSpec(num_layers=16, num_experts=64, k_big=8, k_little=4, hidden_dim=2048, vocab_size=50304,
                  ffn_dim=1024, activation="swiglu", n_heads=16, dtype="bfloat16", seed=0, embed_scale=1.0, pos_encoding="none")

QWEN15_MOE = ModelSpec(num_layers=24, num_experts=60, k_big=4, k_little=2, hidden_dim=2048, vocab_size=151936,
                       ffn_dim=1408, activation="swiglu", n_shared=1, shared_ffn_dim=5632, shared_gate="sigmoid",
                       n_heads=16, dtype="bfloat16", seed=0, embed_scale=1.0, pos_encoding="none")

DEEPSEEK_MOE_16B = ModelSpec(num_layers=27, num_experts=64, k_big=6, k_little=3, hidden_dim=2048, vocab_size=102400,
                             ffn_dim=1408, activation="swiglu", n_shared=2, shared_ffn_dim=1408, n_heads=16,
                             dtype="bfloat16", seed=0, embed_scale=1.0, pos_encoding="none")

MIXTRAL_8X7B = ModelSpec(num_layers=32, num_experts=8, k_big=2, k_little=1, hidden_dim=4096, vocab_size=32000,
                         ffn_dim=14336, activation="swiglu", n_heads=32, n_kv_heads=8, dtype="bfloat16", seed=0,
                         embed_scale=1.0, pos_encoding="none")

PRESETS = {"c1": C1_TINY, "c2": OLMOE, "c3": QWEN15_MOE, "c4": DEEPSEEK_MOE_16B, "c5": MIXTRAL_8X7B}
NAMES = {"c1": "tiny (SPEC.md)", "c2": "OLMoE-1B-7B", "c3": "Qwen1.5-MoE-A2.7B", "c4": "DeepSeek-MoE-16B",
         "c5": "Mixtral-8x7B"}

# the paper's consumer-GPU offload setting (rtx4080.json): 16 GiB cap, 6 GiB reserved
RTX4080_LIKE = HardwareSpec(hbm_capacity=16 * 1024**3, reserved=6 * 1024**3, lookahead_depth=2)


def with_byte_sizes(spec: ModelSpec) -> ModelSpec:
    """Fill expert_bytes / dense_bytes_per_layer from the device layout so
    hbm_expert_slots (config.py:204-218) sees the real sizes."""
    return replace(spec, expert_bytes=spec.device_expert_bytes(),
                   dense_bytes_per_layer=spec.device_dense_bytes_per_layer())
