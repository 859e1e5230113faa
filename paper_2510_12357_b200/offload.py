"""Expert offload runtime: routed experts in pinned host DRAM, a capped HBM
slot pool, cudaMemcpyAsync on a side stream (the paper's offload regime).

This drives libmobile's C++ runtime (mobile_offload_*) with the per-layer
protocol of the reference simulator, `StreamSimulator.run_pass`
(engine.py:121-169):
  (1) at the layer boundary, speculatively issue the plan entries whose window
      opened, dropping stale ones and retrying deferred ones (engine.py:98-119)
  (2) attention
  (3) required request + pin of every selected expert (engine.py:137-145)
  (4) the compute stream waits on their copies (the simulator's "stall")
  (5) expert compute
  (6) unpin (engine.py:152-153)
The little pass and the full-top-k baseline load on demand: their selections
are only known after the layer's router, so the host reads the layer's active
expert list back (one small D2H per layer) before issuing copies
(engine.py:243-244).  The big pass replays the little pass's router logits, so
its whole plan is known up front and copies are issued `lookahead` layers
early (build_mobile_plan, policy.py:86-106).
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from .memory import HbmCache
from .model import ExpertLocation
from .policy import plan_from_targets
from .weights import DeviceWeights
from . import kernels as K


class OffloadRuntime:
    def __init__(self, dw: DeviceWeights, slots: int, lookahead: int = 2):
        if dw.host_experts is None:
            raise ValueError("OffloadRuntime needs DeviceWeights built with experts_on_device=False")
        s = dw.spec
        if slots < s.k_big:
            raise ValueError(f"{slots} expert slots cannot hold one layer's k_big={s.k_big} experts")
        N.reap()  # release handles queued by finalizers before allocating new ones
        self.dw, self.spec = dw, s
        self.L, self.E = s.num_layers, s.num_experts
        self.slots, self.lookahead = slots, lookahead
        dev = dw.device
        self.pool = torch.empty(slots, dw.expert_elems, dtype=dw.wdtype, device=dev)
        self.copy_stream = torch.cuda.Stream(device=dev)
        host = self._host = dw.host_experts
        eb = dw.expert_bytes
        self.h = N.lib.mobile_offload_create(slots, eb, self.pool.data_ptr(), host.data_ptr(), self.E * eb, eb,
                                             self.L, self.E, self.copy_stream.cuda_stream)
        if not self.h:
            raise N.MobileNativeError(N.last_error())
        # slot tables: pinned host rows written by the C++ runtime, device copies read by the kernels
        self.slot_host = torch.zeros(2, self.L, self.E, dtype=torch.int32, pin_memory=True)
        self.slot_dev = torch.zeros(2, self.L, self.E, dtype=torch.int32, device=dev)
        self.active_host = torch.zeros(self.E + 1, dtype=torch.int32, pin_memory=True)
        self.cache = HbmCache(slots, _handle=N.lib.mobile_offload_cache(self.h))
        self.w13_bytes = dw.w13_elems * dw.elem_bytes
        self.pass_log: list = []
        self.fresh = 0

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            N.defer_destroy("mobile_offload_destroy", h, (getattr(self, "pool", None), getattr(self, "_host", None),
                                                           getattr(self, "copy_stream", None)))
            self.h = None

    # ------------------------------------------------------------- runtime ops
    def _location(self, layer: int, row: int) -> ExpertLocation:
        base = self.pool.data_ptr()
        return ExpertLocation(base, base + self.w13_bytes, self.dw.expert_bytes, self.slot_dev[row, layer], self.slots)

    def _require(self, layer: int, experts: list[int], row: int) -> ExpertLocation:
        arr = (C.c_int * len(experts))(*experts)
        issued = C.c_int()
        stream = torch.cuda.current_stream()
        tbl = self.slot_host[row, layer]
        N.check(N.lib.mobile_offload_require(self.h, layer, arr, len(experts), stream.cuda_stream, tbl.data_ptr(),
                                             C.byref(issued)), "offload require")
        self.fresh += issued.value
        self.slot_dev[row, layer].copy_(tbl, non_blocking=True)
        return self._location(layer, row)

    def _release(self, layer: int, experts: list[int]) -> None:
        arr = (C.c_int * len(experts))(*experts)
        N.check(N.lib.mobile_offload_release(self.h, layer, arr, len(experts),
                                             torch.cuda.current_stream().cuda_stream), "offload release")

    def sync_point(self) -> None:
        """The host has just synchronised with the compute stream."""
        N.lib.mobile_offload_sync(self.h)

    def token_end(self) -> None:
        N.check(N.lib.mobile_offload_token_end(self.h), "offload token_end")

    def counters(self) -> tuple[int, int]:
        out = (C.c_longlong * 2)()
        N.lib.mobile_offload_counters(self.h, out)
        return int(out[0]), int(out[1])

    # ------------------------------------------------------------- hooks
    def demand_hook(self, label: str):
        """On-demand loading: the layer's selections are read back after routing."""
        rt = self

        class _Demand:
            def __init__(self):
                self.sel = {}

            def pre(self, layer, r, p):
                # one D2H of the active-expert list; this is the host sync point of the layer
                rt.active_host.copy_(p["active"], non_blocking=True)
                torch.cuda.current_stream().synchronize()
                N.lib.mobile_offload_sync(rt.h)
                n = int(rt.active_host[0])
                experts = rt.active_host[1:1 + n].tolist()
                self.sel[layer] = experts
                return rt._require(layer, experts, 0)

            def post(self, layer):
                rt._release(layer, self.sel.pop(layer))

        return _Demand()

    def plan_hooks(self, router_states: torch.Tensor, k_big: int):
        """Planned (replayed) big pass: targets = top_k(h_s[l], k_big) for every
        layer, issue windows max(0, l - lookahead) (policy.py:86-106)."""
        idx, _ = K.topk_rows(router_states.contiguous(), k_big)
        targets = idx.cpu().tolist()  # one D2H for the whole pass
        plan = plan_from_targets(targets, self.lookahead)
        rt = self
        waiting = list(plan.entries)

        def layer_hook(layer):  # engine.py:98-119 _issue_window
            nonlocal waiting
            kept = []
            st = C.c_int()
            for i, e in enumerate(waiting):
                if e.earliest_issue_layer > layer:
                    kept.extend(waiting[i:])
                    break
                if e.expert.layer < layer or e.after_routing:
                    continue
                rc = N.lib.mobile_offload_prefetch(rt.h, e.expert.layer, e.expert.expert, C.byref(st))
                if rc == N.ERR_DEFERRED:
                    kept.append(e)
                else:
                    N.check(rc, "offload prefetch")
            waiting = kept

        class _Planned:
            def pre(self, layer, r, p):
                return rt._require(layer, targets[layer], 1)

            def post(self, layer):
                rt._release(layer, targets[layer])

        return _Planned(), layer_hook
