"""Fallback rule and prefetch planning (drop-in for moesim.policy).

`should_fallback` (policy.py:69-79) and the per-layer top-k of
`build_mobile_plan` (policy.py:86-106) run on the device (libmobile
probs-check and row top-k kernels); the plan's issue windows and ordering are
host bookkeeping over those indices.  The modeled pre-gating baseline
(`build_pregated_plan`) is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from .spec import ExpertId


@dataclass(frozen=True)
class PlanEntry:
    expert: ExpertId
    earliest_issue_layer: int
    after_routing: bool


@dataclass
class PrefetchPlan:
    """targets[l] = experts layer l executes; entries sorted by (issue, layer, expert)."""

    targets: list[list[ExpertId]]
    entries: list[PlanEntry]

    @property
    def num_layers(self) -> int:
        return len(self.targets)


def _dev():
    if not torch.cuda.is_available():
        from ._native import MobileNativeError
        raise MobileNativeError("no CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def should_fallback(probs, gamma: float) -> bool:
    """True iff max(probs) <= gamma (strict > accepts); |sum - 1| > 1e-4 raises."""
    a = np.ascontiguousarray(np.asarray(probs, dtype=np.float64).reshape(-1))
    total, mx = K.probs_check(torch.as_tensor(a).to(_dev())).cpu().tolist()
    if abs(total - 1.0) > 1e-4:
        raise ValueError(f"probability vector sums to {total}, expected 1 within 1e-4")
    return bool(mx <= gamma)


def _order(entries: list[PlanEntry]) -> list[PlanEntry]:
    return sorted(entries, key=lambda e: (e.earliest_issue_layer, e.expert.layer, e.expert.expert))


def plan_from_targets(targets: list[list[int]], lookahead: int) -> PrefetchPlan:
    """Plan for known per-layer targets: every entry issuable `lookahead` layers early."""
    tg = [[ExpertId(l, int(e)) for e in row] for l, row in enumerate(targets)]
    entries = [PlanEntry(x, max(0, l - lookahead), False) for l, row in enumerate(tg) for x in row]
    return PrefetchPlan(tg, _order(entries))


def build_mobile_plan(router_states, k_big: int, lookahead: int) -> PrefetchPlan:
    """All-layers-up-front plan from the recorded little-pass logits (policy.py:86-106)."""
    if lookahead < 1:
        raise ValueError(f"lookahead must be >= 1, got {lookahead}")
    if isinstance(router_states, torch.Tensor) and router_states.is_cuda:
        states = router_states
        if states.dim() != 2:
            raise ValueError(f"router states must be 2-D (layers x experts), got shape {tuple(states.shape)}")
    else:
        a = np.asarray(router_states, dtype=float)
        if a.ndim != 2:
            raise ValueError(f"router states must be 2-D (layers x experts), got shape {a.shape}")
        states = torch.as_tensor(np.ascontiguousarray(a)).to(_dev())
    if k_big > states.shape[1]:
        raise ValueError(f"k ({k_big}) exceeds number of experts ({states.shape[1]})")
    idx, flags = K.topk_rows(states, k_big)
    if int(flags.item()) & 1:
        raise ValueError("router logits must be finite")
    return plan_from_targets(idx.cpu().tolist(), lookahead)


def on_demand_selection(selection: list[list[ExpertId]]) -> PrefetchPlan:
    """Every expert loads at its own layer, after routing (policy.py:109-116)."""
    entries = []
    for layer, chosen in enumerate(selection):
        if not chosen:
            raise ValueError(f"layer {layer} has an empty expert selection")
        entries += [PlanEntry(c, layer, True) for c in chosen]
    return PrefetchPlan([list(s) for s in selection], _order(entries))


def selections_from_logits(layers, k: int) -> list[list[ExpertId]]:
    """Per-layer top-k ExpertIds of an (L, E) logit matrix (engine.py:76-81), on the device."""
    a = np.asarray(layers, dtype=float)
    idx, flags = K.topk_rows(torch.as_tensor(np.ascontiguousarray(a)).to(_dev()), k)
    if int(flags.item()) & 1:
        raise ValueError("router logits must be finite")
    return [[ExpertId(l, int(e)) for e in row] for l, row in enumerate(idx.cpu().tolist())]


def fallback_flags_from_confidence(records, gamma: float) -> list[bool]:
    """engine.py:266-268: strict `> gamma` accepts."""
    return [rec.confidence <= gamma for rec in records]


def injected_fallback_flags(n_tokens: int, ratio: float) -> list[bool]:
    """Evenly spaced flags with exactly floor(n * ratio) fallbacks (engine.py:271-277)."""
    if not (0.0 <= ratio <= 1.0):
        raise ValueError(f"fallback ratio outside [0, 1]: {ratio}")
    eps = 1e-9
    return [int((i + 1) * ratio + eps) > int(i * ratio + eps) for i in range(n_tokens)]


def build_pregated_plan(*args, **kwargs):
    """policy.py:119-153 (the modelled pre-gating competitor) is out of scope
    (DESIGN.md §5): the name exists so `moesim` code importing it loads."""
    raise NotImplementedError("build_pregated_plan: the pre-gating baseline (policy.py:119-153) is out of scope")
