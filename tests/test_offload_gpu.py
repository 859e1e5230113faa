"""Expert offload runtime (pinned host store + HBM slot cache + copy stream) on the GPU.

The offloaded decode must produce exactly the resident decode's tokens and
selections (same kernels, same weights -- only the expert addresses differ),
under a cache small enough to force evictions, deferrals and deadlock stalls.
"""
import numpy as np
import pytest
import torch

from tests.helpers import QWEN_MINI, matched

pytestmark = pytest.mark.gpu


def _offloaded(spec_kw, dtype):
    from paper_2510_12357_b200.model import DeviceModel
    from paper_2510_12357_b200.weights import DeviceWeights
    o, ms, dm = matched(spec_kw, dtype)
    dw = dm.dw
    host = dw.experts.cpu().pin_memory()
    dw2 = DeviceWeights(ms, dw.device, experts_on_device=False)
    for name in ("embed", "qkv", "o", "router", "shared", "head"):
        setattr(dw2, name, getattr(dw, name))
    dw2.host_experts = host
    return o, ms, dm, DeviceModel(dw2)


@pytest.mark.parametrize("slots", [4, 6, 24])
@pytest.mark.parametrize("full", [False, True])
def test_offload_decode_equals_resident(cuda_ok, slots, full):
    from paper_2510_12357_b200 import PolicySpec
    from paper_2510_12357_b200.decode import MobileGenerator
    from paper_2510_12357_b200.offload import OffloadRuntime
    o, ms, dm_res, dm_off = _offloaded(QWEN_MINI, "bfloat16")
    flags = [bool(i % 3 == 1) for i in range(14)]
    # prefill touches up to min(E, ctx * k_big) experts per layer at once; keep
    # the context short enough for the smallest caches
    prompt = [5, 9] if slots < 12 else [5, 9, 100, 7, 33]
    ref = MobileGenerator(dm_res, 64)
    t_ref, d_ref = ref.generate(prompt, PolicySpec(), 14, fallback_flags=flags, stop_at_eos=False, full=full)
    rt = OffloadRuntime(dm_off.dw, slots, lookahead=1)
    gen = MobileGenerator(dm_off, 64, runtime=rt)
    t_off, d_off = gen.generate(prompt, PolicySpec(), 14, fallback_flags=flags, stop_at_eos=False, full=full)
    assert t_off == t_ref
    for a, b in zip(d_off, d_ref):
        assert a.accepted_by == b.accepted_by
        assert a.little_selections == b.little_selections and a.big_selections == b.big_selections
    st = rt.cache.stats
    nbytes, transfers = rt.counters()
    assert transfers == st.issued >= rt.fresh  # required misses + speculative prefetches
    assert nbytes == transfers * dm_off.dw.expert_bytes
    assert len(rt.cache) <= slots
    if slots < ms.num_layers * ms.num_experts:
        assert st.evictions > 0


def test_offload_rejects_tiny_cache(cuda_ok):
    from paper_2510_12357_b200.offload import OffloadRuntime
    o, ms, dm_res, dm_off = _offloaded(QWEN_MINI, "bfloat16")
    with pytest.raises(ValueError):
        OffloadRuntime(dm_off.dw, ms.k_big - 1)
