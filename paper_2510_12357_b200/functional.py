"""Drop-in for `moesim.toymoe` (toymoe.py:1-303) running on the B200.

Same names, signatures, result types and error messages: `build_model`,
`forward`, `little_forward`, `big_forward`, `full_forward`, `generate`,
`top_k`, `softmax`, `ToyMoE`, `ForwardResult`, `TokenDecision`.  Results come
back as host NumPy arrays (fp64 probabilities, router logits) as the
reference's tests expect; all arithmetic runs in libmobile kernels on the GPU
(fp32 compute, fp64 final softmax).  There is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import kernels as K
from .model import DecodeSession, DeviceModel
from .spec import SAMPLING_TEMPERATURE, ModelSpec, PolicySpec
from .weights import DeviceWeights, HostWeights, check_toy_limits, init_host_weights

ACCEPTED_LITTLE = "Little"
ACCEPTED_BIG = "BigFallback"
LOGIT_SCALE = 24.0


def _device():
    if not torch.cuda.is_available():
        raise N.MobileNativeError("no CUDA device: the MoBiLE layer runs only on the GPU (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass
class ToyMoE:
    """Weights (reference layout, host fp64) + their device copy (lazy)."""

    spec: ModelSpec
    embed: np.ndarray
    attn_q: np.ndarray
    attn_k: np.ndarray
    attn_v: np.ndarray
    attn_o: np.ndarray
    router: np.ndarray
    expert_in: np.ndarray
    expert_out: np.ndarray
    head: np.ndarray
    host: HostWeights = field(repr=False, default=None)
    _dm: DeviceModel | None = field(repr=False, default=None)

    @property
    def device_model(self) -> DeviceModel:
        if self._dm is None:
            self._dm = DeviceModel(DeviceWeights.from_host(self.spec, self.host, _device()))
        return self._dm


@dataclass
class ForwardResult:
    probs: np.ndarray  # (V,)
    router_states: np.ndarray  # (L, E)
    selections: list[list[int]]


@dataclass
class TokenDecision:
    token: int
    accepted_by: str
    confidence: float
    little_selections: list[list[int]]
    big_selections: list[list[int]] | None = None
    router_states: np.ndarray | None = None


def _finite_or_raise(flags: torch.Tensor) -> None:
    f = int(flags.item())
    if f & 1:
        raise ValueError("router logits must be finite")


def top_k(logits, k: int) -> list[int]:
    """Indices of the k largest logits, descending, ties to the lower index (device kernel)."""
    a = np.asarray(logits)
    E = a.shape[-1]
    if k > E:
        raise ValueError(f"k ({k}) exceeds number of experts ({E})")
    rows = torch.as_tensor(np.ascontiguousarray(a.reshape(1, E), dtype=np.float64)).to(_device())
    idx, flags = K.topk_rows(rows, k)
    _finite_or_raise(flags)
    return [int(i) for i in idx[0].cpu().tolist()]


def softmax(x) -> np.ndarray:
    """toymoe.py:91-94 (fp64 device kernel)."""
    a = np.asarray(x, dtype=np.float64)
    t = torch.as_tensor(np.ascontiguousarray(a.reshape(1, -1))).to(_device())
    return K.softmax_rows(t, torch.float64)[0].cpu().numpy().reshape(a.shape)


def build_model(spec: ModelSpec) -> ToyMoE:
    """Seeded weights in the reference's draw order (toymoe.py:97-126)."""
    spec.validate()
    check_toy_limits(spec)
    hw = init_host_weights(spec)
    return ToyMoE(spec, hw.embed, hw.attn_q, hw.attn_k, hw.attn_v, hw.attn_o, hw.router, hw.expert_in,
                  hw.expert_out, hw.head, host=hw)


def forward(model: ToyMoE, tokens: list[int], k: int, replay_states=None, reuse_gates: bool = False) -> ForwardResult:
    """toymoe.py:143-210 on the device."""
    spec = model.spec
    if not tokens:
        raise ValueError("token sequence is empty")
    for t in tokens:
        if not (0 <= t < spec.vocab_size):
            raise ValueError(f"token {t} outside vocab [0, {spec.vocab_size})")
    if k > spec.num_experts:
        raise ValueError(f"k ({k}) exceeds number of experts ({spec.num_experts})")
    if replay_states is not None:
        replay_states = np.asarray(replay_states, dtype=float)
        if replay_states.shape != (spec.num_layers, spec.num_experts):
            raise ValueError(f"router states shape {replay_states.shape} does not match "
                             f"(num_layers, num_experts) = ({spec.num_layers}, {spec.num_experts})")
        if not np.all(np.isfinite(replay_states)):
            raise ValueError("router logits must be finite")
    probs, states, sels, flags = model.device_model.forward_recompute(list(tokens), k, replay_states, reuse_gates)
    _finite_or_raise(flags)
    return ForwardResult(probs=probs.cpu().numpy(), router_states=states.double().cpu().numpy(),
                         selections=[[int(e) for e in row] for row in sels.cpu().tolist()])


def little_forward(model: ToyMoE, tokens: list[int]) -> ForwardResult:
    return forward(model, tokens, model.spec.k_little)


def big_forward(model: ToyMoE, tokens: list[int], router_states, reuse_gates: bool = False) -> ForwardResult:
    return forward(model, tokens, model.spec.k_big, replay_states=router_states, reuse_gates=reuse_gates)


def full_forward(model: ToyMoE, tokens: list[int]) -> ForwardResult:
    return forward(model, tokens, model.spec.k_big)


def _sample(probs: np.ndarray, policy: PolicySpec, rng: np.random.Generator) -> int:
    """toymoe.py:239-243 (host-side draw from the device probabilities)."""
    if policy.sampling == SAMPLING_TEMPERATURE:
        logp = np.log(probs) / policy.temperature
        z = np.exp(logp - logp.max())
        return int(rng.choice(len(probs), p=z / z.sum()))
    return int(np.argmax(probs))


def _should_fallback_host(probs: np.ndarray, gamma: float) -> bool:
    from .policy import should_fallback
    return should_fallback(probs, gamma)


def generate(model: ToyMoE, prompt: list[int], policy: PolicySpec, max_len: int,
             record_router_states: bool = False):
    """Algorithm 1 (toymoe.py:246-303): little pass, confidence test, replayed big pass."""
    if not prompt:
        raise ValueError("prompt is empty")
    if max_len < 1:
        raise ValueError(f"max_len must be >= 1, got {max_len}")
    policy.validate()
    rng = np.random.default_rng(policy.sampling_seed)
    tokens = list(prompt)
    decisions: list[TokenDecision] = []
    while len(decisions) < max_len:
        little = little_forward(model, tokens)
        confidence = float(little.probs.max())
        if _should_fallback_host(little.probs, policy.gamma):
            big = big_forward(model, tokens, little.router_states, reuse_gates=policy.reuse_little_gates)
            token = _sample(big.probs, policy, rng)
            decisions.append(TokenDecision(token, ACCEPTED_BIG, confidence, little.selections, big.selections,
                                           little.router_states))
        else:
            token = _sample(little.probs, policy, rng)
            decisions.append(TokenDecision(token, ACCEPTED_LITTLE, confidence, little.selections, None,
                                           little.router_states if record_router_states else None))
        tokens.append(token)
        if token == model.spec.eos_token:
            break
    return tokens, decisions
