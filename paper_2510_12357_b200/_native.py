"""ctypes binding of libmobile.so (include/mobile.h).

The CUDA extension is the product path: if it is missing or fails to load,
importing the package's compute modules raises -- there is no CPU fallback.
Status codes are mapped back to the reference's exception types and message
substrings (toymoe.py:83-86, memory.py:137-144, memory.py:174-177).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("MOBILE_LIB", _PKG / "libmobile.so"))

OK, ERR_INVALID, ERR_K_EXCEEDS, ERR_NONFINITE, ERR_CUDA, ERR_DEADLOCK, ERR_DEFERRED, ERR_UNSUPPORTED, ERR_NOT_FOUND = range(9)
F32, BF16, F64 = 0, 1, 2
ACT_RELU, ACT_SWIGLU = 0, 1
GATE_SELECTED_SOFTMAX, GATE_SOFTMAX_ALL = 0, 1
STATUS_NAMES = {0: "hit", 1: "in_flight", 2: "issued"}


class MobileNativeError(RuntimeError):
    """CUDA / unsupported-shape failure inside libmobile."""


class CapacityDeadlock(RuntimeError):
    """A required expert load found every cache slot pinned or in flight (memory.py:25-26)."""


class mobile_sg_group(C.Structure):
    _fields_ = [("w_base", C.c_void_p), ("stride", C.c_longlong), ("slot", C.c_void_p), ("x", C.c_void_p),
                ("x_div", C.c_int), ("offsets", C.c_void_p), ("pairs", C.c_void_p), ("active", C.c_void_p),
                ("dense_T", C.c_int), ("max_active", C.c_int), ("K", C.c_int), ("rows", C.c_int),
                ("out", C.c_void_p), ("residual", C.c_void_p), ("epi", C.c_int), ("prefetch", C.c_int)]


class mobile_channel(C.Structure):
    _fields_ = [("t_xfer", C.c_double), ("busy_until", C.c_double), ("transfers_issued", C.c_longlong)]


class mobile_dp_model(C.Structure):
    """include/mobile.h mobile_dp_model (persistent decode pass)."""
    _fields_ = [(n, C.c_int) for n in ("B", "L", "d", "H", "V", "E", "k", "n_shared", "n_gate", "ffn", "shared_ffn",
                                       "activation", "gate_norm", "reuse_gates", "w_dtype", "max_len", "offload",
                                       "Hkv")] + [
        ("logit_scale", C.c_float), ("gamma", C.c_float),
        ("qkv", C.c_void_p), ("o", C.c_void_p), ("router", C.c_void_p), ("shared", C.c_void_p),
        ("shared_stride", C.c_longlong), ("shared_w2_offset", C.c_longlong), ("experts", C.c_void_p),
        ("expert_layer_stride", C.c_longlong), ("expert_stride", C.c_longlong), ("expert_w2_offset", C.c_longlong),
        ("slot_table", C.c_void_p), ("head", C.c_void_p), ("embed", C.c_void_p), ("pe", C.c_void_p),
        ("tok", C.c_void_p), ("pos", C.c_void_p), ("kc", C.c_void_p), ("vc", C.c_void_p),
        ("x", C.c_void_p), ("xa", C.c_void_p), ("q", C.c_void_p), ("att", C.c_void_p),
        ("U", C.c_void_p), ("Us", C.c_void_p), ("Y", C.c_void_p), ("Ys", C.c_void_p),
        ("states", C.c_void_p), ("extra", C.c_void_p), ("replay", C.c_void_p), ("idx_out", C.c_void_p),
        ("gates_out", C.c_void_p), ("active_out", C.c_void_p), ("head_logits", C.c_void_p), ("conf", C.c_void_p),
        ("argmax", C.c_void_p), ("fallback", C.c_void_p), ("flags", C.c_void_p)]


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} not found: build the CUDA extension first "
            f"(python -m paper_2510_12357_b200.build or __graft_entry__.build()); "
            f"there is no CPU fallback")
    return C.CDLL(str(LIB_PATH))


lib = _load()

P, I32, I64, F, D, SZ = C.c_void_p, C.c_int, C.c_longlong, C.c_float, C.c_double, C.c_size_t
_SIGS = {
    "mobile_version": ([], I32),
    "mobile_last_error": ([], C.c_char_p),
    "mobile_num_sms": ([], I32),
    "mobile_router_topk": ([P, P, P, I32, I32, I32, I32, I32, I32, P, P, P, I32, I32, P, P, P, P, P, P, P, P, P],
                           I32),
    "mobile_router_topk_pf": ([P, P, P, I32, I32, I32, I32, I32, I32, P, P, P, I32, I32, P, P, P, P, P, P, P, P,
                               P, I64, I64, P], I32),
    "mobile_topk_rows": ([P, I32, I32, I32, I32, P, P, P], I32),
    "mobile_head_ws_bytes": ([I32, I32], SZ),
    "mobile_head_confidence": ([P, P, I32, I32, I32, I32, F, F, P, P, P, P, P, P], I32),
    "mobile_softmax_rows": ([P, I32, P, I32, I32, I32, P], I32),
    "mobile_logits_confidence": ([P, I32, I32, F, F, P, P, P, P], I32),
    "mobile_probs_check": ([P, I32, I32, P, P], I32),
    "mobile_permute": ([P, P, I32, I32, I32, P, P, P, P], I32),
    "mobile_combine": ([P, P, P, P, I32, I32, I32, P, I32, P, P, P, P], I32),
    "mobile_grouped_gemm": ([P, I32, I32, P, I64, I32, I32, P, P, P, I32, I32, I32, I32, P, P, I32, I32, P, P], I32),
    "mobile_gather_rows_bf16": ([P, P, I32, I32, I32, P, P], I32),
    "mobile_gather_bf16": ([P, P, I32, I32, I32, P, P], I32),
    "mobile_gather_ln_bf16": ([P, P, I32, I32, I32, P, P], I32),
    "mobile_ep_mailbox_bytes": ([I32, I32, I32], SZ),
    "mobile_ep_mailbox_create": ([I32, I32, I32, P], I32),
    "mobile_ep_mailbox_destroy": ([P], I32),
    "mobile_ep_ipc_handle": ([P, P], I32),
    "mobile_ep_ipc_open": ([P, P], I32),
    "mobile_ep_ipc_close": ([P], I32),
    "mobile_ep_dispatch": ([P, P, P, I32, I32, I32, P, P, P, I32, I32, I32, C.c_uint, P, I32, P, P, P, P], I32),
    "mobile_ep_wait": ([P, I32, I32, I32, I32, C.c_uint, P, P, P, P], I32),
    "mobile_ep_return": ([P, P, P, I32, I32, I32, I32, C.c_uint, P, P], I32),
    "mobile_ep_advance": ([P, P], I32),
    "mobile_ep_collect": ([P, P, I32, I32, I32, I32, P, P], I32),
    "mobile_stream_gemv": ([P, I32, I32, I32, P], I32),
    "mobile_stream_head_ws_bytes": ([], SZ),
    "mobile_stream_head": ([P, I32, I32, P, I32, I32, F, F, P, P, P, P, P, P], I32),
    "mobile_dense_gemv": ([P, I32, I32, I32, P, I32, I32, P, P, P], I32),
    "mobile_attn_decode": ([P, P, P, P, I32, I32, I32, I32, P, P], I32),
    "mobile_attn_split_ws": ([I32, I32, I32, I32, P, P], I32),
    "mobile_attn_decode_ws": ([P, P, P, P, I32, I32, I32, I32, I32, P, P, P, I32, I32, P], I32),
    "mobile_embed": ([P, P, P, P, I32, I32, P, P, P], I32),
    "mobile_advance": ([P, I32, P, P, P], I32),
    "mobile_memcpy_async": ([P, P, SZ, P], I32),
    "mobile_cache_create": ([I32], P),
    "mobile_cache_destroy": ([P], None),
    "mobile_cache_request": ([P, I32, I32, D, I32, P, D, P, P, P], I32),
    "mobile_cache_pin": ([P, I32, I32], I32),
    "mobile_cache_unpin": ([P, I32, I32], I32),
    "mobile_cache_token_end": ([P], I32),
    "mobile_cache_evict_lru": ([P, I32, D, P, P], I32),
    "mobile_cache_size": ([P], I32),
    "mobile_cache_contains": ([P, I32, I32], I32),
    "mobile_cache_lookup": ([P, I32, I32, P, P], I32),
    "mobile_cache_set_ready": ([P, I32, I32, D], I32),
    "mobile_cache_entries": ([P, P, I32], I32),
    "mobile_cache_stats": ([P, P], I32),
    "mobile_offload_create": ([I32, I64, P, P, I64, I64, I32, I32, P], P),
    "mobile_offload_destroy": ([P], None),
    "mobile_offload_require": ([P, I32, P, I32, P, P, P], I32),
    "mobile_offload_prefetch": ([P, I32, I32, P], I32),
    "mobile_offload_release": ([P, I32, P, I32, P], I32),
    "mobile_offload_sync": ([P], I32),
    "mobile_offload_token_end": ([P], I32),
    "mobile_offload_cache": ([P], P),
    "mobile_offload_counters": ([P, P], I32),
    "mobile_offload_run_pass": ([P, P, I32, P, I32, P, P, I32, P, P, I64, I32, P], I32),
    "mobile_dp_create": ([P, P], I32),
    "mobile_dp_destroy": ([P], None),
    "mobile_dp_num_segments": ([P], I32),
    "mobile_dp_info": ([P, P], I32),
    "mobile_dp_launch": ([P, I32, P], I32),
    "mobile_dp_set_trace": ([P, P], I32),
    "mobile_dp_set_events": ([P, P], I32),
    "mobile_dp_diag": ([P, P], I32),
    "mobile_dp_run_offload_pass": ([P, P, I32, P, I32, I32, P, P], I32),
    "mobile_offload_zs_enable": ([P, P, P, P, P], I32),
    "mobile_offload_zs_require": ([P, I32, P, I32, P, P, P, P], I32),
    "mobile_offload_zs_prefetch": ([P, I32, I32, P], I32),
    "mobile_offload_zs_release": ([P, I32, P, I32, I64], I32),
    "mobile_offload_zs_base": ([P], P),
}
EXPORTED = tuple(_SIGS)
for _name, (_args, _ret) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _ret


# Finalizers run wherever the GC fires -- possibly inside another engine's
# CUDA-graph capture, where the cudaFree / cudaFreeHost / stream destroys of a
# native handle would invalidate that capture.  Destroys are queued instead
# and run at the next safe point (`reap`, called before graph captures and
# handle creation), with the torch objects the handle points into kept alive.
_deferred: list = []


def defer_destroy(fn_name: str, handle, keepalive=()) -> None:
    _deferred.append((fn_name, handle, tuple(keepalive)))


def reap() -> None:
    """Run queued native destroys (not during a capture: callers ensure it)."""
    if not _deferred:
        return
    import torch
    if torch.cuda.is_available():
        torch.cuda.synchronize()
    while _deferred:
        fn_name, handle, _keep = _deferred.pop(0)
        getattr(lib, fn_name)(handle)


def last_error() -> str:
    return (lib.mobile_last_error() or b"").decode()


def check(status: int, what: str = "") -> int:
    """Raise the reference-compatible exception for a non-OK status."""
    if status == OK:
        return status
    msg = last_error()
    if status in (ERR_INVALID, ERR_K_EXCEEDS, ERR_NONFINITE, ERR_NOT_FOUND):
        raise ValueError(msg or what)
    if status == ERR_DEADLOCK:
        raise CapacityDeadlock(msg)
    raise MobileNativeError(f"{what}: {msg} (status {status})")


def ptr(t) -> int | None:
    """Raw device/host pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()
