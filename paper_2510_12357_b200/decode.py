"""KV-cached MoBiLE decode (Algorithm 1 with one position per step).

Per generated token: the little pass (k_little experts per layer, own
routing) runs on the new position; the head kernel yields the confidence and
the fallback flag (max p <= gamma) on the device; a fallback token re-runs the
position at k_big with every layer's final-position selection replayed from
the little pass's recorded router logits (toymoe.py:272-278) and its K/V rows
replace the little pass's.  The context part of the prompt is prefilled at
`prefill_k` (k_big by default).  `fallback_flags` overrides the confidence
rule per decision (engine.injected_fallback_flags), which is how benchmarks
pin the fallback ratio r.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels as K
from .functional import ACCEPTED_BIG, ACCEPTED_LITTLE
from .model import DecodeSession, DeviceModel
from .spec import PolicySpec


@dataclass
class KVDecision:
    token: int
    accepted_by: str
    confidence: float
    little_selections: list
    big_selections: list | None = None
    router_states: np.ndarray | None = None


@dataclass
class DecodeStats:
    tokens: int = 0
    fallbacks: int = 0
    little_passes: int = 0
    big_passes: int = 0
    per_token_ms: list = field(default_factory=list)


class MobileGenerator:
    """Batch-1 MoBiLE generator over a DecodeSession (device-resident experts
    unless `runtime` -- an offload.OffloadRuntime -- supplies them)."""

    def __init__(self, dm: DeviceModel, max_len: int, prefill_k: int | None = None, runtime=None):
        self.dm, self.spec = dm, dm.spec
        self.max_len = max_len
        self.prefill_k = self.spec.k_big if prefill_k is None else prefill_k
        self.runtime = runtime
        dev = dm.device
        s = self.spec
        self.k_l = torch.full((1,), s.k_little, dtype=torch.int32, device=dev)
        self.k_b = torch.full((1,), s.k_big, dtype=torch.int32, device=dev)
        self.one = torch.ones(1, dtype=torch.uint8, device=dev)
        self.ws = dm.stream_head_ws()
        self.head_out = dict(conf=torch.empty(1, device=dev), argmax=torch.empty(1, device=dev, dtype=torch.int32),
                             fallback=torch.empty(1, device=dev, dtype=torch.uint8))
        self.stats = DecodeStats()
        self.timer = None  # optional kernel timer (bench roofline)

    def _head(self, x_last, gamma):
        import torch.nn.functional as Fn
        x_ln = Fn.layer_norm(x_last, (self.spec.hidden_dim,), eps=1e-5).contiguous()
        return K.stream_head(x_ln, self.dm.dw.head, gamma, self.spec.logit_scale, ws=self.ws, out=self.head_out)

    def start(self, prompt: list[int]) -> DecodeSession:
        dm, s = self.dm, self.spec
        sess = DecodeSession(dm, 1, self.max_len)
        ctx = list(prompt[:-1])
        if ctx:
            t = torch.tensor([ctx], dtype=torch.long, device=dm.device)
            k = torch.full((len(ctx),), self.prefill_k, dtype=torch.int32, device=dm.device)
            hook = self.runtime.demand_hook("prefill") if self.runtime else None
            sess.run(t, k, self.prefill_k, expert_hook=hook)
            if self.runtime:
                self.runtime.token_end()
        return sess

    def step_full(self, sess: DecodeSession, last: int, record: bool = False) -> KVDecision:
        """Full-top-k baseline step: one k_big pass with its own routing,
        experts loaded on demand (engine.simulate_full_stream, on_demand plan)."""
        s, dev = self.spec, self.dm.device
        tok = torch.tensor([[last]], dtype=torch.long, device=dev)
        rt = self.runtime
        hook = rt.demand_hook("full") if rt else None
        x, states, idx = sess.run(tok, self.k_b, s.k_big, advance=False, expert_hook=hook, timer=self.timer)
        out = self._head(x, 1.0)
        token = int(out["argmax"].item())
        if rt:
            rt.sync_point()
            rt.token_end()
        sess.pos += 1
        self.stats.tokens += 1
        self.stats.big_passes += 1
        return KVDecision(token, ACCEPTED_BIG, float(out["conf"].item()) if record else float("nan"),
                          [], idx[:, 0].cpu().tolist() if record else None, None)

    def step(self, sess: DecodeSession, last: int, policy: PolicySpec, forced_fallback: bool | None = None,
             record: bool = False) -> KVDecision:
        s, dev = self.spec, self.dm.device
        tok = torch.tensor([[last]], dtype=torch.long, device=dev)
        rt = self.runtime
        hook = rt.demand_hook("little") if rt else None
        x, states, idx_l = sess.run(tok, self.k_l, s.k_little, advance=False, expert_hook=hook, timer=self.timer)
        out = self._head(x, policy.gamma)
        self.stats.little_passes += 1
        fb_dev = out["fallback"]
        if forced_fallback is None:
            fb = bool(fb_dev.item())
        else:
            fb = bool(forced_fallback)
        conf = float(out["conf"].item()) if record else float("nan")
        if rt:
            torch.cuda.current_stream().synchronize()
            rt.sync_point()
        if fb:
            if rt:
                plan_hook, layer_hook = rt.plan_hooks(states[:, 0], s.k_big)
            else:
                plan_hook = layer_hook = None
            xb, _, idx_b = sess.run(tok, self.k_b, s.k_big, replay=states, replay_mask=self.one,
                                    reuse_gates=policy.reuse_little_gates, advance=False,
                                    expert_hook=plan_hook, layer_hook=layer_hook, timer=self.timer)
            out = self._head(xb, policy.gamma)
            self.stats.big_passes += 1
            self.stats.fallbacks += 1
        token = int(out["argmax"].item())
        if rt:
            rt.token_end()
        sess.pos += 1
        self.stats.tokens += 1
        if record:
            lsel = idx_l[:, 0].cpu().tolist()
            return KVDecision(token, ACCEPTED_BIG if fb else ACCEPTED_LITTLE, conf, lsel,
                              idx_b[:, 0].cpu().tolist() if fb else None,
                              states[:, 0].double().cpu().numpy() if fb else None)
        return KVDecision(token, ACCEPTED_BIG if fb else ACCEPTED_LITTLE, conf, [], None, None)

    def generate(self, prompt: list[int], policy: PolicySpec, max_new: int, fallback_flags=None,
                 record: bool = True, stop_at_eos: bool = True, full: bool = False):
        if not prompt:
            raise ValueError("prompt is empty")
        if max_new < 1:
            raise ValueError(f"max_len must be >= 1, got {max_new}")
        if len(prompt) + max_new > self.max_len:
            raise ValueError(f"prompt + max_len exceeds the session capacity {self.max_len}")
        sess = self.start(prompt)
        tokens, decisions = list(prompt), []
        while len(decisions) < max_new:
            forced = None if fallback_flags is None else bool(fallback_flags[len(decisions)])
            if full:
                d = self.step_full(sess, tokens[-1], record)
            else:
                d = self.step(sess, tokens[-1], policy, forced, record)
            decisions.append(d)
            tokens.append(d.token)
            if stop_at_eos and d.token == self.spec.eos_token:
                break
        return tokens, decisions
