"""B200-native MoBiLE mixture-of-big-little-experts MoE layer.

Drop-in for the hot path of the reference package `moesim`
(/root/reference/pkg/src/moesim): the same public names for model/layer
construction, the big/little routing and fallback options, and the
forward/generate entry points, the plan builder and the expert cache -- with
the arithmetic in hand-written sm_100a CUDA kernels (libmobile.so, C ABI in
include/mobile.h).  Importing this package loads libmobile.so and fails
loudly if it is missing: there is no CPU fallback.
"""

from . import _native  # noqa: F401  (loads libmobile.so; raises if absent)
from ._native import CapacityDeadlock, MobileNativeError
from .functional import (
    ACCEPTED_BIG,
    ACCEPTED_LITTLE,
    LOGIT_SCALE,
    ForwardResult,
    TokenDecision,
    ToyMoE,
    big_forward,
    build_model,
    forward,
    full_forward,
    generate,
    little_forward,
    softmax,
    top_k,
)
from .memory import HIT, IN_FLIGHT, ISSUED, CacheStats, HbmCache, RequestResult, TransferChannel
from .model import DecodeSession, DeviceModel, MoBiLEMoE
from .policy import (
    PlanEntry,
    PrefetchPlan,
    build_mobile_plan,
    fallback_flags_from_confidence,
    injected_fallback_flags,
    on_demand_selection,
    selections_from_logits,
    should_fallback,
)
from .spec import (
    ConfigError,
    CostTable,
    ExpertId,
    HardwareSpec,
    ModelSpec,
    PolicySpec,
    data_path,
    derive_costs,
    hbm_expert_slots,
    load_config_file,
    parse_bytes,
)
from .weights import DeviceWeights, HostWeights, init_host_weights

__version__ = "0.1.0"
