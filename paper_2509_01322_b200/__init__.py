"""B200-native ScMoE layer (LongCat-Flash shortcut-connected MoE with
zero-computation experts) behind the reference's operator API.

The numeric work is done by ``libscmoe.so`` (hand-written sm_100a CUDA: exact
fp32 router, permutation, tcgen05 grouped GEMM, combine, bias controller),
reached through its C ABI (``include/scmoe.h``).  This module mirrors the
reference's C++ API (moelab, /root/reference/proj/include/moelab) with the
same names, argument meanings and error types, so parity tests read like the
reference's own tests:

    RouterState            router.hpp:20-62
    RoutingDecision        router.hpp:64-87
    select_topk_row        router.hpp:90-104
    route_from_probs       router.hpp:107-130
    route_topk             router.hpp:133-141
    accumulate_counters    router.hpp:144-150
    bias_update            router.hpp:155-176
    simulate_bias_control  router.hpp:349-369
    GammaMode, ExpertBank  blocks.hpp:185-213
    moe_forward            blocks.hpp:372-394
    scmoe_layer_forward    model.hpp:394-400 (MoE branch of build_layer)

There is no CPU implementation here: when the CUDA library or a B200 is
missing every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import threading
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libscmoe.so")


# ---- error taxonomy (common.hpp:11-33) -------------------------------------
class MoelabError(RuntimeError):
    pass


class DimensionError(MoelabError):
    pass


class ParameterError(MoelabError, ValueError):
    pass


class ConfigError(MoelabError):
    pass


class StateError(MoelabError):
    pass


class DeviceError(MoelabError):
    """CUDA / driver failure (no reference equivalent)."""


_ERRORS = {1: ConfigError, 2: DimensionError, 3: StateError, 4: ParameterError, 5: DeviceError,
           6: MoelabError}

PREC_F32_EXACT = 0
PREC_BF16 = 1
PREC_F64_EXACT = 2


class GammaMode(enum.IntEnum):
    """blocks.hpp:185"""
    FfnOnly = 0
    All = 1
    Off = 2


# ---- library loading -------------------------------------------------------
_lib = None
_lib_lock = threading.Lock()

_P = C.c_void_p
_SZ = C.c_size_t
_U64 = C.c_uint64
_PROTOS = {
    "scmoe_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "scmoe_ctx_destroy": (C.c_int, [_P]),
    "scmoe_last_error": (C.c_char_p, [_P]),
    "scmoe_set_stream": (C.c_int, [_P, _P]),
    "scmoe_get_stream": (_P, [_P]),
    "scmoe_synchronize": (C.c_int, [_P]),
    "scmoe_kernel_launches": (_U64, [_P]),
    "scmoe_version": (C.c_char_p, []),
    "scmoe_device_alloc": (C.c_int, [_P, _SZ, C.POINTER(_P)]),
    "scmoe_device_free": (C.c_int, [_P, _P]),
    "scmoe_copy_h2d": (C.c_int, [_P, _P, _P, _SZ]),
    "scmoe_copy_d2h": (C.c_int, [_P, _P, _P, _SZ]),
    "scmoe_router_create": (C.c_int, [_P, _SZ, _SZ, _SZ, _SZ, _SZ, C.c_double, C.c_double,
                                      C.POINTER(_P)]),
    "scmoe_router_destroy": (C.c_int, [_P, _P]),
    "scmoe_router_set_weights_host": (C.c_int, [_P, _P, _P]),
    "scmoe_router_set_weights": (C.c_int, [_P, _P, _P]),
    "scmoe_router_set_bias_host": (C.c_int, [_P, _P, _P]),
    "scmoe_router_get_bias_host": (C.c_int, [_P, _P, _P]),
    "scmoe_router_set_mu": (C.c_int, [_P, _P, C.c_double, C.c_double]),
    "scmoe_router_get_mu": (C.c_int, [_P, _P, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "scmoe_router_get_counters_host": (C.c_int, [_P, _P, _P, C.POINTER(_U64)]),
    "scmoe_router_set_counters_host": (C.c_int, [_P, _P, _P, _U64]),
    "scmoe_router_counters_dev": (_P, [_P]),
    "scmoe_router_bias_dev": (_P, [_P]),
    "scmoe_route_topk": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _P, _P]),
    "scmoe_route_topk_host": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _P, _P]),
    "scmoe_route_from_probs_f32": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _P]),
    "scmoe_route_from_probs_f64": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _P]),
    "scmoe_route_from_probs_f32_host": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _P]),
    "scmoe_route_from_probs_f64_host": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _P]),
    "scmoe_accumulate_counters": (C.c_int, [_P, _P, _P, _SZ]),
    "scmoe_route_topk_f64": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _P, _P, _P]),
    "scmoe_route_topk_f64_host": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _P, _P, _P]),
    "scmoe_debug_exp": (C.c_int, [_P, _P, _P, _SZ]),
    "scmoe_bank_set_expert_f64": (C.c_int, [_P, _P, _SZ, _P, _P]),
    "scmoe_bank_set_expert_f64_host": (C.c_int, [_P, _P, _SZ, _P, _P]),
    "scmoe_moe_forward_f64": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _SZ, _SZ, C.c_int, _P, _P]),
    "scmoe_moe_forward_f64_host": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _SZ, _SZ, C.c_int, _P,
                                             _P]),
    "scmoe_routing_stats": (C.c_int, [_P, _P, _P, _SZ, _SZ, _SZ, _SZ, _SZ, _SZ, _P, _P, _P, _P]),
    "scmoe_routing_stats_host": (C.c_int, [_P, _P, _P, _SZ, _SZ, _SZ, _SZ, _SZ, _SZ, _P, _P, _P,
                                           _P]),
    "scmoe_accumulate_counters_host": (C.c_int, [_P, _P, _P, _SZ]),
    "scmoe_bias_update": (C.c_int, [_P, _P, _P]),
    "scmoe_bank_create": (C.c_int, [_P, _SZ, _SZ, _SZ, C.c_int, _SZ, C.c_int, C.POINTER(_P)]),
    "scmoe_bank_destroy": (C.c_int, [_P, _P]),
    "scmoe_bank_set_expert_host": (C.c_int, [_P, _P, _SZ, _P, _P]),
    "scmoe_bank_set_expert": (C.c_int, [_P, _P, _SZ, _P, _P]),
    "scmoe_bank_init_uniform": (C.c_int, [_P, _P, _U64, _U64, C.c_double]),
    "scmoe_bank_gamma_ffn": (C.c_double, [_P]),
    "scmoe_bank_gamma_zero": (C.c_double, [_P]),
    "scmoe_bank_device_bytes": (_SZ, [_P]),
    "scmoe_moe_forward": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _SZ, _SZ, C.c_int, _P, _P]),
    "scmoe_moe_forward_host": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _SZ, _SZ, C.c_int, _P, _P]),
    "scmoe_rmsnorm": (C.c_int, [_P, _P, _P, _SZ, _SZ, C.c_float, _P]),
    "scmoe_layer_forward": (C.c_int, [_P, _P, _P, _P, _P, _P, _SZ, C.c_int, _P, _P, _P, _P]),
    "scmoe_layer_forward_host": (C.c_int, [_P, _P, _P, _P, _P, _P, _SZ, C.c_int, _P, _P, _P,
                                           _P]),
    "scmoe_layer_forward_batches": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _P, _SZ, C.c_int, _P, _P,
                                              _P, _P]),
    "scmoe_dense_ffn": (C.c_int, [_P, _P, _P, _P, _SZ, _P]),
    "scmoe_ep_put_rows": (C.c_int, [_P, _P, _SZ, _P, _P, _SZ, _P, _P, _P, _P, C.c_int]),
    "scmoe_moe_rows_to": (C.c_int, [_P, _P, _P, _P, C.c_int, _SZ, _P]),
    "scmoe_ctx_set_sm_budget": (C.c_int, [_P, C.c_int, C.c_int]),
    "scmoe_ctx_set_overlapped": (C.c_int, [_P, C.c_int]),
    "scmoe_layer_forward_host_batches": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _P, _SZ, C.c_int, _P,
                                                   _P, _P, _P]),
    "scmoe_bank_init_uniform_shard": (C.c_int, [_P, _P, _U64, _U64, C.c_double, _SZ]),
    "scmoe_rmsnorm_route": (C.c_int, [_P, _P, _P, _P, _SZ, _P, _P, _P, _P, _P]),
    "scmoe_ep_plan": (C.c_int, [_P, _P, _SZ, _SZ, _SZ, _SZ, C.c_int, _P, _P, _P, _P]),
    "scmoe_gather_rows_bf16": (C.c_int, [_P, _P, _SZ, _P, _SZ, _P]),
    "scmoe_permutation": (C.c_int, [_P, _P, _SZ, _SZ, _SZ, _SZ, _P, _P]),
    "scmoe_mla_set_precision": (C.c_int, [_P, _P, C.c_int]),
    "scmoe_ep_unique_id_bytes": (_SZ, []),
    "scmoe_ep_unique_id": (C.c_int, [_P]),
    "scmoe_ep_create": (C.c_int, [_P, C.c_int, C.c_int, _P, _SZ, _SZ, _SZ, _SZ, _SZ, _SZ,
                                  C.POINTER(_P)]),
    "scmoe_ep_destroy": (C.c_int, [_P]),
    "scmoe_ep_capacity_rows": (_SZ, [_P]),
    "scmoe_ep_kernel_launches": (_U64, [_P]),
    "scmoe_ep_set_comm": (C.c_int, [_P, C.c_int]),
    "scmoe_ep_set_dense_reserve": (C.c_int, [_P, C.c_int]),
    "scmoe_ep_layer_forward": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _SZ, C.c_int, _P, _P, _P,
                                         _P]),
    "scmoe_ep_layer_forward_batches": (C.c_int, [_P, _P, _P, _SZ, _P, _P, _P, _SZ, C.c_int,
                                                 C.c_int, _P, _P, _P, _P]),
    "scmoe_ep_controller_step": (C.c_int, [_P, _P, _P, _SZ, C.c_int, _P]),
    "scmoe_ep_count_matrix_host": (C.c_int, [_P, _P]),
    "scmoe_moe_rows": (C.c_int, [_P, _P, _P, _P, C.c_int, _SZ, _P]),
    "scmoe_combine_rows": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _SZ, _SZ, _SZ, C.c_int, _P,
                                     _P]),
    "scmoe_rng_stream_seed": (_U64, [_U64, _U64]),
    "scmoe_rng_fill_normal_host": (None, [_U64, _U64, _SZ, _P, C.c_int]),
    "scmoe_rng_fill_uniform": (C.c_int, [_P, _U64, _U64, _SZ, C.c_double, _P]),
    "scmoe_profile_enable": (C.c_int, [_P, C.c_int]),
    "scmoe_profile_flush": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "scmoe_profile_span": (C.c_int, [_P, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)]),
    "scmoe_profile_entry": (C.c_int, [_P, C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_double),
                                      C.POINTER(_U64)]),
    "scmoe_debug_expf": (C.c_int, [_P, _P, _P, _SZ]),
    "scmoe_debug_expf_range": (C.c_int, [_P, C.c_uint32, _P, _SZ]),
    "scmoe_mla_create": (C.c_int, [_P] + [_SZ] * 6 + [C.c_double, C.c_int, _P]),
    "scmoe_mla_destroy": (C.c_int, [_P, _P]),
    "scmoe_mla_set_weight_host": (C.c_int, [_P, _P, C.c_int, _P]),
    "scmoe_mla_set_weight": (C.c_int, [_P, _P, C.c_int, _P]),
    "scmoe_mla_forward": (C.c_int, [_P, _P, _P, _SZ, _SZ, _P]),
    "scmoe_mla_forward_host": (C.c_int, [_P, _P, _P, _SZ, _SZ, _P]),
    "scmoe_mla_cache_create": (C.c_int, [_P, _P, _SZ, _P]),
    "scmoe_mla_cache_destroy": (C.c_int, [_P, _P]),
    "scmoe_mla_cache_length": (C.c_int, [_P, _P, C.POINTER(_SZ)]),
    "scmoe_mla_cache_read_host": (C.c_int, [_P, _P, _P, _P, _P]),
    "scmoe_mla_infer_step": (C.c_int, [_P, _P, _P, _P, _SZ, _P]),
    "scmoe_mla_infer_step_host": (C.c_int, [_P, _P, _P, _P, _SZ, _P]),
    "scmoe_layer_full_forward": (C.c_int, [_P] * 11 + [_SZ, _SZ, C.c_int, C.c_int] + [_P] * 6),
}


def exported_symbols() -> list[str]:
    return sorted(_PROTOS)


def lib():
    """The loaded libscmoe.so.  Raises if the CUDA extension was not built."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2509_01322_b200.build` "
                    "(there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in _PROTOS.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_P)


class Context:
    """One CUDA device + stream + workspace (scmoe_ctx).  Not thread-safe:
    use one per thread, as the C ABI requires."""

    def __init__(self, device: int = 0):
        self._h = _P()
        self._check(lib().scmoe_ctx_create(device, C.byref(self._h)), ctx=False)

    def _check(self, rc: int, ctx: bool = True):
        if rc != 0:
            msg = lib().scmoe_last_error(self._h).decode() if ctx and self._h else "scmoe call failed"
            raise _ERRORS.get(rc, MoelabError)(msg)

    @property
    def handle(self):
        return self._h

    def synchronize(self):
        self._check(lib().scmoe_synchronize(self._h))

    def set_stream(self, stream_ptr: int | None):
        self._check(lib().scmoe_set_stream(self._h, stream_ptr))

    def kernel_launches(self) -> int:
        return int(lib().scmoe_kernel_launches(self._h))

    def set_overlapped(self, on: bool = True):
        """Router launches use the kernel that co-resides with a GEMM on another
        stream (for callers that pipeline batches themselves)."""
        self._check(lib().scmoe_ctx_set_overlapped(self._h, int(on)))

    def set_sm_budget(self, router_sms: int = 0, gemm_sms: int = 0):
        """Cap the CTAs of the persistent router / grouped GEMM (0 = all SMs)."""
        self._check(lib().scmoe_ctx_set_sm_budget(self._h, router_sms, gemm_sms))

    def profile(self, on: bool = True):
        self._check(lib().scmoe_profile_enable(self._h, int(on)))

    def profile_flush(self) -> dict:
        """{stage: (total_ms, launches)} since the last flush (syncs the stream)."""
        n = C.c_int()
        self._check(lib().scmoe_profile_flush(self._h, C.byref(n)))
        out = {}
        for i in range(n.value):
            name, ms, cnt = C.c_char_p(), C.c_double(), _U64()
            self._check(lib().scmoe_profile_entry(self._h, i, C.byref(name), C.byref(ms),
                                                  C.byref(cnt)))
            out[name.value.decode()] = (ms.value, int(cnt.value))
        return out

    def profile_spans(self) -> list:
        """[(stage, start_ms, end_ms)] of the last profile_flush(), issue order."""
        out, i = [], 0
        while True:
            name, a, b = C.c_char_p(), C.c_double(), C.c_double()
            if lib().scmoe_profile_span(self._h, i, C.byref(name), C.byref(a), C.byref(b)) != 0:
                return out
            out.append((name.value.decode(), a.value, b.value))
            i += 1

    def close(self):
        if self._h:
            lib().scmoe_ctx_destroy(self._h)
            self._h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: dict[int, Context] = {}


def default_context() -> Context:
    tid = threading.get_ident()
    c = _default_ctx.get(tid)
    if c is None:
        c = Context(int(os.environ.get("SCMOE_DEVICE", "0")))
        _default_ctx[tid] = c
    return c


# ---- router ------------------------------------------------------------------
class RouterState:
    """RouterState<float> (router.hpp:20-62): projection w [d, N+Z], selection
    bias b (zero for identity experts), PID constants and load counters.

    The device copy (scmoe_router) is created lazily and re-synchronised when
    the host fields change (``w``/``b``/counters are plain numpy arrays, as
    the reference's are plain vectors)."""

    def __init__(self, w: Optional[np.ndarray], n_ffn: int, n_zero: int, top_k: int,
                 k_expected: int, mu: float, mu_decay: float):
        # S = float (the hot path) or S = double (RouterState<double>): kept as given
        dt = np.float64 if (w is not None and np.asarray(w).dtype == np.float64) else np.float32
        self.w = None if w is None else np.ascontiguousarray(w, dtype=dt)
        self.n_ffn, self.n_zero, self.top_k, self.k_expected = n_ffn, n_zero, top_k, k_expected
        self.mu, self.mu_decay = float(mu), float(mu_decay)
        self.b = np.zeros(n_ffn + n_zero, dtype=np.float64)
        self.tokens_routed = np.zeros(n_ffn + n_zero, dtype=np.uint64)
        self.tokens_seen = 0
        self.validate()
        self._dev = None
        self._dev_key = None

    def n_experts(self) -> int:
        return self.n_ffn + self.n_zero

    def validate(self):
        """router.hpp:50-61 (same checks, same order)."""
        if self.top_k > self.n_experts():
            raise ConfigError("router: top_k exceeds expert count")
        if self.k_expected < 1 or self.k_expected > self.top_k:
            raise ConfigError("router: need 1 <= k_expected <= top_k")
        if self.n_zero > 0 and self.k_expected >= self.top_k:
            raise ConfigError("router: k_expected must be < top_k when zero experts exist")
        if self.n_zero < self.top_k - self.k_expected:
            raise ConfigError("router: too few zero experts to absorb top_k - k_expected slack")
        if self.mu < 0.0:
            raise ConfigError("router: mu must be >= 0")
        if np.any(np.asarray(self.b)[self.n_ffn:] != 0.0):
            raise ConfigError("router: zero-expert bias must stay 0")

    # Device mirror ----------------------------------------------------------
    def device(self, ctx: Context):
        """Returns the scmoe_router handle with w/b/mu/counters uploaded.  The
        mirror is recreated when the context or the shape fields change, and
        the weights re-uploaded when any of their bytes change (a CRC32 over
        the whole buffer, no copy: ~2 ms for the 18.9 MB LongCat W_r)."""
        import zlib
        L = lib()
        E = self.n_experts()
        d = 0 if self.w is None else self.w.shape[0]
        shape = (d, self.n_ffn, self.n_zero, self.top_k, self.k_expected)
        if self._dev is None or self._dev[0] is not ctx or self._dev[2] != shape:
            self.close()
            h = _P()
            ctx._check(L.scmoe_router_create(ctx.handle, d, self.n_ffn, self.n_zero, self.top_k,
                                             self.k_expected, self.mu, self.mu_decay, C.byref(h)))
            self._dev = (ctx, h, shape)
            self._dev_key = None
        h = self._dev[1]
        wkey = None if self.w is None else (
            id(self.w), self.w.ctypes.data, self.w.shape, self.w.dtype.str,
            zlib.crc32(memoryview(np.ascontiguousarray(self.w)).cast("B")))
        if self.w is not None and (self._dev_key is None or self._dev_key != wkey):
            if self.w.shape != (d, E):
                raise DimensionError("route: router weights must be [d_model, N+Z]")
            w32 = np.ascontiguousarray(self.w, dtype=np.float32)
            ctx._check(L.scmoe_router_set_weights_host(ctx.handle, h, _ptr(w32)))
            self._dev_key = wkey
        b = np.ascontiguousarray(self.b, dtype=np.float64)
        ctx._check(L.scmoe_router_set_bias_host(ctx.handle, h, _ptr(b)))
        ctx._check(L.scmoe_router_set_mu(ctx.handle, h, self.mu, self.mu_decay))
        tr = np.ascontiguousarray(self.tokens_routed, dtype=np.uint64)
        ctx._check(L.scmoe_router_set_counters_host(ctx.handle, h, _ptr(tr), int(self.tokens_seen)))
        return h

    def close(self):
        """Destroys the device mirror (recreated on the next use)."""
        dev, self._dev = getattr(self, "_dev", None), None
        if dev is not None and dev[0].handle:
            lib().scmoe_router_destroy(dev[0].handle, dev[1])

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def pull(self, ctx: Context):
        """Copies b / mu / counters back from the device mirror."""
        L = lib()
        h = self._dev[1]
        b = np.empty(self.n_experts(), dtype=np.float64)
        ctx._check(L.scmoe_router_get_bias_host(ctx.handle, h, _ptr(b)))
        mu, dec = C.c_double(), C.c_double()
        ctx._check(L.scmoe_router_get_mu(ctx.handle, h, C.byref(mu), C.byref(dec)))
        tr = np.empty(self.n_experts(), dtype=np.uint64)
        seen = _U64()
        ctx._check(L.scmoe_router_get_counters_host(ctx.handle, h, _ptr(tr), C.byref(seen)))
        self.b, self.mu, self.tokens_routed, self.tokens_seen = b, mu.value, tr, int(seen.value)


@dataclass
class RoutingDecision:
    """router.hpp:64-87"""
    top_k: int = 0
    n_ffn: int = 0
    indices: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    gates: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))
    ffn_count: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))

    def tokens(self) -> int:
        return len(self.ffn_count)

    def mean_ffn(self) -> float:
        if len(self.ffn_count) == 0:
            return 0.0
        s = 0.0
        for c in self.ffn_count.tolist():
            s += c
        return s / len(self.ffn_count)

    def std_ffn(self) -> float:
        if len(self.ffn_count) == 0:
            return 0.0
        m = self.mean_ffn()
        s = 0.0
        for c in self.ffn_count.tolist():
            s += (c - m) * (c - m)
        return float(np.sqrt(s / len(self.ffn_count)))


def _as2d(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    if a.ndim != 2:
        raise DimensionError("expected a 2-d tensor")
    return a


def route_topk(x: np.ndarray, state: RouterState, probs_out: Optional[list] = None,
               ctx: Optional[Context] = None) -> RoutingDecision:
    """router.hpp:133-141.  x [T, d] fp32 (or fp64 with a float64 RouterState:
    RouterState<double>).  If ``probs_out`` is a list, the probabilities
    [T, N+Z] are appended to it (the reference's Tensor* out)."""
    ctx = ctx or default_context()
    state.validate()
    f64 = state.w is not None and state.w.dtype == np.float64
    x = _as2d(x, np.float64 if f64 else np.float32)
    if state.w is None:
        raise DimensionError("matmul: operands must be 2-d")
    if x.shape[1] != state.w.shape[0]:
        raise DimensionError("matmul: inner dims disagree")
    T, K, E = x.shape[0], state.top_k, state.n_experts()
    h = state.device(ctx)
    idx = np.empty(T * K, np.uint32)
    gates = np.empty(T * K, np.float64)
    cnt = np.empty(T, np.uint32)
    probs = np.empty((T, E), np.float64 if f64 else np.float32) if probs_out is not None else None
    if f64:
        ctx._check(lib().scmoe_route_topk_f64_host(ctx.handle, h, _ptr(x), T, _ptr(state.w),
                                                   _ptr(idx), _ptr(gates), _ptr(cnt),
                                                   _ptr(probs)))
    else:
        ctx._check(lib().scmoe_route_topk_host(ctx.handle, h, _ptr(x), T, _ptr(idx), _ptr(gates),
                                               _ptr(cnt), _ptr(probs)))
    if probs_out is not None:
        probs_out.append(probs)
    return RoutingDecision(K, state.n_ffn, idx, gates, cnt)


def route_from_probs(probs: np.ndarray, state: RouterState,
                     ctx: Optional[Context] = None) -> RoutingDecision:
    """router.hpp:107-130; float32 or float64 probabilities [T, N+Z]."""
    ctx = ctx or default_context()
    state.validate()
    probs = np.asarray(probs)
    dt = np.float64 if probs.dtype == np.float64 else np.float32
    probs = _as2d(probs, dt)
    if probs.shape[1] != state.n_experts():
        raise DimensionError("route: probs width mismatch")
    T, K = probs.shape[0], state.top_k
    h = state.device(ctx)
    idx = np.empty(T * K, np.uint32)
    gates = np.empty(T * K, np.float64)
    cnt = np.empty(T, np.uint32)
    fn = lib().scmoe_route_from_probs_f64_host if dt == np.float64 else \
        lib().scmoe_route_from_probs_f32_host
    ctx._check(fn(ctx.handle, h, _ptr(probs), T, _ptr(idx), _ptr(gates), _ptr(cnt)))
    return RoutingDecision(K, state.n_ffn, idx, gates, cnt)


def select_topk_row(probs_row: np.ndarray, bias: Sequence[float], n_experts: int, k: int,
                    ctx: Optional[Context] = None) -> np.ndarray:
    """router.hpp:90-104: indices of the k largest double(p)+b, ties to the
    lowest index.  Runs the device top-k kernel on a one-token batch."""
    ctx = ctx or default_context()
    dt = np.float64 if np.asarray(probs_row).dtype == np.float64 else np.float32
    p = np.ascontiguousarray(np.asarray(probs_row, dtype=dt)[:n_experts]).reshape(1, n_experts)
    # A scratch router with n_ffn = n_experts (no zero experts) carries the bias.
    st = RouterState(None, n_experts, 0, k, k, 0.0, 1.0)
    st.b = np.ascontiguousarray(np.asarray(bias, dtype=np.float64)[:n_experts])
    return route_from_probs(p, st, ctx).indices


def accumulate_counters(state: RouterState, d: RoutingDecision, ctx: Optional[Context] = None):
    """router.hpp:144-150 (slot-counted, zero experts included), on the device."""
    ctx = ctx or default_context()
    idx = np.ascontiguousarray(d.indices, np.uint32)
    h = state.device(ctx)
    ctx._check(lib().scmoe_accumulate_counters_host(ctx.handle, h, _ptr(idx), d.tokens()))
    state.pull(ctx)


def routing_stats(d: RoutingDecision, n_zero: int, k_expected: int, lb_groups: Optional[int] = None,
                  ctx: Optional[Context] = None) -> dict:
    """Per-layer routing statistics from a device histogram:
    mean / std of activated FFN experts (router.hpp:73-86), per-expert slot
    load (stats.hpp:64-67) and, with lb_groups, the LB group frequencies
    (router.hpp:193-216).  Bitwise equal to the reference."""
    ctx = ctx or default_context()
    idx = np.ascontiguousarray(d.indices, np.uint32)
    cnt = np.ascontiguousarray(d.ffn_count, np.uint32)
    T, E = d.tokens(), d.n_ffn + n_zero
    mean, std = C.c_double(), C.c_double()
    load = np.empty(E, np.float64)
    lb = np.empty(lb_groups + (1 if n_zero else 0), np.float64) if lb_groups else None
    ctx._check(lib().scmoe_routing_stats_host(ctx.handle, _ptr(idx), _ptr(cnt), T, d.top_k,
                                              d.n_ffn, n_zero, k_expected, lb_groups or 0,
                                              C.byref(mean), C.byref(std), _ptr(load),
                                              _ptr(lb) if lb is not None else None))
    out = {"mean_activated_ffn": mean.value, "std_activated_ffn": std.value,
           "per_expert_load": load}
    if lb is not None:
        out["lb_group_frequencies"] = lb
    return out


def bias_update(state: RouterState, ctx: Optional[Context] = None) -> np.ndarray:
    """router.hpp:155-176 on the device; returns the applied deltas."""
    ctx = ctx or default_context()
    if state.tokens_seen == 0:
        raise StateError("bias_update: empty batch")
    h = state.device(ctx)
    delta = np.empty(state.n_experts(), np.float64)
    ctx._check(lib().scmoe_bias_update(ctx.handle, h, _ptr(delta)))
    state.pull(ctx)
    return delta


@dataclass
class BiasControlTrace:
    """router.hpp:343-347"""
    mean_ffn: list = field(default_factory=list)
    std_ffn: list = field(default_factory=list)
    bias_history: list = field(default_factory=list)


def fill_normal(seed: int, n: int, first: int = 0, threads: int = 8) -> np.ndarray:
    """x[i] = (float) CounterRng(seed).normal_at(first + i)  (rng.hpp:51-55)."""
    out = np.empty(n, np.float32)
    lib().scmoe_rng_fill_normal_host(seed, first, n, _ptr(out), threads)
    return out


def stream_seed(seed: int, sid: int) -> int:
    """CounterRng(seed).stream(sid).seed()  (rng.hpp:35)."""
    return int(lib().scmoe_rng_stream_seed(seed, sid))


def simulate_bias_control(state: RouterState, d_model: int, batch_tokens: int, steps: int,
                          rng_seed: int, keep_bias_history: bool = False,
                          ctx: Optional[Context] = None) -> BiasControlTrace:
    """router.hpp:349-369: per step fresh x = normal_at(i) of rng.stream(step),
    route (device), count (device), record mean/std ffn, bias_update (device)."""
    ctx = ctx or default_context()
    L = lib()
    tr = BiasControlTrace()
    h = state.device(ctx)
    T, K = batch_tokens, state.top_k
    idx = np.empty(T * K, np.uint32)
    gates = np.empty(T * K, np.float64)
    cnt = np.empty(T, np.uint32)
    for step in range(steps):
        x = fill_normal(stream_seed(rng_seed, step), T * d_model)
        ctx._check(L.scmoe_route_topk_host(ctx.handle, h, _ptr(x), T, _ptr(idx), _ptr(gates),
                                           _ptr(cnt), None))
        ctx._check(L.scmoe_accumulate_counters_host(ctx.handle, h, _ptr(idx), T))
        d = RoutingDecision(K, state.n_ffn, idx, gates, cnt)
        tr.mean_ffn.append(d.mean_ffn())
        tr.std_ffn.append(d.std_ffn())
        ctx._check(L.scmoe_bias_update(ctx.handle, h, None))
        if keep_bias_history:
            state.pull(ctx)
            tr.bias_history.append(state.b.copy())
    state.pull(ctx)
    return tr


# ---- expert bank / MoE -----------------------------------------------------------
class ExpertBank:
    """ExpertBank<float> (blocks.hpp:203-213): per-expert w_in [d, I] and
    w_out [I, d], segmentation factor m and GammaMode.  ``precision`` selects
    the exact fp32 kernels (bitwise equal to the reference) or the bf16
    tcgen05 path.  Weights are uploaded once (device residency) and
    re-uploaded only through set_expert / invalidate."""

    def __init__(self, w_in: Sequence[np.ndarray], w_out: Sequence[np.ndarray], m: int = 1,
                 gamma_mode: GammaMode = GammaMode.FfnOnly, precision: int = PREC_F32_EXACT):
        # PREC_F64_EXACT is ExpertBank<double> (weights kept in double)
        dt = np.float64 if precision == PREC_F64_EXACT else np.float32
        self.w_in = [np.ascontiguousarray(w, dt) for w in w_in]
        self.w_out = [np.ascontiguousarray(w, dt) for w in w_out]
        self.m, self.gamma_mode, self.precision = m, GammaMode(gamma_mode), precision
        if m < 1:
            raise ParameterError("variance_gamma: m must be >= 1")
        self._dev = None

    def n_experts(self) -> int:
        return len(self.w_in)

    def gamma_ffn(self) -> float:
        return 1.0 if self.gamma_mode == GammaMode.Off else float(self.m)

    def gamma_zero(self) -> float:
        return float(self.m) if self.gamma_mode == GammaMode.All else 1.0

    def invalidate(self):
        """Drops the device copy: the next use re-uploads the host weights
        (call after changing w_in / w_out in place)."""
        self.close()

    def close(self):
        dev, self._dev = getattr(self, "_dev", None), None
        if dev is not None and dev[0].handle:
            lib().scmoe_bank_destroy(dev[0].handle, dev[1])

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def device(self, ctx: Context):
        if self._dev is not None and self._dev[0] is ctx:
            return self._dev[1]
        self.close()
        n = self.n_experts()
        d, I = self.w_in[0].shape if n else (0, 0)
        h = _P()
        ctx._check(lib().scmoe_bank_create(ctx.handle, n, d, I, self.precision, self.m,
                                           int(self.gamma_mode), C.byref(h)))
        try:
            for e in range(n):
                if self.w_in[e].shape != (d, I) or self.w_out[e].shape != (I, d):
                    raise DimensionError("moe_block: expert weight shapes disagree")
                setter = (lib().scmoe_bank_set_expert_f64_host if self.precision == PREC_F64_EXACT
                          else lib().scmoe_bank_set_expert_host)
                ctx._check(setter(ctx.handle, h, e, _ptr(self.w_in[e]), _ptr(self.w_out[e])))
        except Exception:
            lib().scmoe_bank_destroy(ctx.handle, h)
            raise
        self._dev = (ctx, h)
        return h


def moe_forward(x: np.ndarray, d: RoutingDecision, bank: ExpertBank, n_zero: int,
                renormalize: bool = False, residual: Optional[np.ndarray] = None,
                ctx: Optional[Context] = None) -> np.ndarray:
    """blocks.hpp:372-394 (+ optional renormalisation and fused residual).
    An fp64 bank (PREC_F64_EXACT) computes moe_forward<double> on fp64 x."""
    ctx = ctx or default_context()
    f64 = bank.precision == PREC_F64_EXACT
    dt = np.float64 if f64 else np.float32
    x = _as2d(x, dt)
    T, dm = x.shape
    K = d.top_k
    idx = np.ascontiguousarray(d.indices, np.uint32)
    gates = np.ascontiguousarray(d.gates, np.float64)
    e_total = bank.n_experts() + n_zero
    if idx.size and int(idx.max()) >= e_total:
        raise StateError("moe_forward: expert index out of range")
    if d.n_ffn != bank.n_experts():
        raise DimensionError("moe_block: decision/bank FFN count mismatch")
    if idx.size != T * K or gates.size != T * K:
        raise DimensionError("moe_combine: slot map size mismatch")
    h = bank.device(ctx)
    out = np.empty((T, dm), dt)
    res = None if residual is None else _as2d(residual, dt)
    fn = lib().scmoe_moe_forward_f64_host if f64 else lib().scmoe_moe_forward_host
    ctx._check(fn(ctx.handle, h, _ptr(x), T, _ptr(idx), _ptr(gates), K, n_zero, int(renormalize),
                  _ptr(res), _ptr(out)))
    return out


def scmoe_layer_forward(a1: np.ndarray, a3: np.ndarray, gain: Optional[np.ndarray],
                        state: RouterState, bank: ExpertBank, renormalize: bool = False,
                        ctx: Optional[Context] = None):
    """MoE branch of Model::build_layer (model.hpp:394-400):
    out = a3 + moe_block(rmsnorm(a1, gain), softmax(rmsnorm(a1) W_r), ...).
    Returns (out, RoutingDecision)."""
    ctx = ctx or default_context()
    a1 = _as2d(a1, np.float32)
    a3 = _as2d(a3, np.float32)
    T, dm = a1.shape
    K = state.top_k
    hr = state.device(ctx)
    hb = bank.device(ctx)
    g = None if gain is None else np.ascontiguousarray(gain, np.float32)
    idx = np.empty(T * K, np.uint32)
    gates = np.empty(T * K, np.float64)
    cnt = np.empty(T, np.uint32)
    out = np.empty((T, dm), np.float32)
    ctx._check(lib().scmoe_layer_forward_host(ctx.handle, hr, hb, _ptr(a1), _ptr(a3), _ptr(g), T,
                                              int(renormalize), _ptr(idx), _ptr(gates), _ptr(cnt),
                                              _ptr(out)))
    return out, RoutingDecision(K, state.n_ffn, idx, gates, cnt)


__all__ = [
    "ConfigError", "DimensionError", "StateError", "ParameterError", "DeviceError", "GammaMode",
    "RouterState", "RoutingDecision", "select_topk_row", "route_from_probs", "route_topk",
    "accumulate_counters", "bias_update", "simulate_bias_control", "BiasControlTrace",
    "ExpertBank", "moe_forward", "scmoe_layer_forward", "Context", "default_context", "lib",
    "fill_normal", "stream_seed", "PREC_F32_EXACT", "PREC_BF16",
]
