"""ctypes access to the parity checkers (TEST INFRASTRUCTURE).

    ORC  oracle/liboracle.so          C restatement (oracle/scmoe_oracle.c)
    REF  oracle/_ref/libmoelab_ref.so the reference's own templates (ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may use this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORC_PATH = os.path.join(ORACLE_DIR, "liboracle.so")
REF_PATH = os.path.join(ORACLE_DIR, "_ref", "libmoelab_ref.so")

_P = C.c_void_p
_SZ = C.c_size_t
_U64 = C.c_uint64
_D = C.c_double

ERR = {0: None, 1: "ConfigError", 2: "DimensionError", 3: "StateError", 4: "ParameterError"}


def build_oracle():
    if not os.path.exists(ORC_PATH) or (
            os.path.exists("/root/reference") and not os.path.exists(REF_PATH)):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def _load(path, protos):
    L = C.CDLL(path)
    for name, (res, args) in protos.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


_ORC_PROTOS = {
    "orc_hash2": (_U64, [_U64, _U64]),
    "orc_stream_seed": (_U64, [_U64, _U64]),
    "orc_normal_at": (_D, [_U64, _U64]),
    "orc_fill_normal_f32": (None, [_U64, _U64, _U64, _P]),
    "orc_fill_normal_f64": (None, [_U64, _U64, _U64, _P]),
    "orc_seeded_uniform_f32": (C.c_int, [_U64, _U64, _U64, _D, _P]),
    "orc_seeded_tn_f64": (C.c_int, [_U64, _U64, _D, _P]),
    "orc_seeded_tn_f32": (C.c_int, [_U64, _U64, _D, _P]),
    "orc_mm_f32": (None, [_P, _P, _P, _SZ, _SZ, _SZ]),
    "orc_mm_f64": (None, [_P, _P, _P, _SZ, _SZ, _SZ]),
    "orc_softmax_rows_f32": (None, [_P, _P, _SZ, _SZ]),
    "orc_softmax_rows_f64": (None, [_P, _P, _SZ, _SZ]),
    "orc_rmsnorm_f32": (None, [_P, _P, _SZ, _SZ, C.c_float, _P]),
    "orc_expf": (C.c_float, [C.c_float]),
    "orc_expf_range": (None, [C.c_uint32, _SZ, _P]),
    "orc_router_validate": (C.c_int, [_SZ, _SZ, _SZ, _SZ, _D, _P]),
    "orc_select_topk_row_f32": (None, [_P, _P, _SZ, _SZ, _P]),
    "orc_select_topk_row_f64": (None, [_P, _P, _SZ, _SZ, _P]),
    "orc_route_from_probs_f32": (C.c_int, [_P, _SZ, _SZ, _SZ, _SZ, _SZ, _D, _P, _P, _P, _P]),
    "orc_route_from_probs_f64": (C.c_int, [_P, _SZ, _SZ, _SZ, _SZ, _SZ, _D, _P, _P, _P, _P]),
    "orc_route_topk_f32": (C.c_int, [_P, _SZ, _SZ, _P, _SZ, _SZ, _SZ, _SZ, _D, _P, _P, _P, _P,
                                     _P]),
    "orc_route_topk_f64": (C.c_int, [_P, _SZ, _SZ, _P, _SZ, _SZ, _SZ, _SZ, _D, _P, _P, _P, _P,
                                     _P]),
    "orc_accumulate_counters": (None, [_P, _SZ, _SZ, _P, _P]),
    "orc_routing_stats": (C.c_int, [_P, _P, _SZ, _SZ, _SZ, _SZ, _SZ, _SZ, _P, _P, _P, _P]),
    "orc_bias_update": (C.c_int, [_SZ, _SZ, _SZ, _SZ, _P, _D, _P, _P, _P, _P]),
    "orc_moe_forward_f32": (C.c_int, [_P, _SZ, _SZ, _P, _P, _SZ, _SZ, _SZ, _P, _P, _SZ, _D, _D,
                                      C.c_int, _P]),
    "orc_moe_forward_f64": (C.c_int, [_P, _SZ, _SZ, _P, _P, _SZ, _SZ, _SZ, _P, _P, _SZ, _D, _D,
                                      C.c_int, _P]),
    "orc_permutation": (None, [_P, _SZ, _SZ, _SZ, _SZ, _P, _P]),
    "orc_moe_forward_streamed_f32": (C.c_int, [_P, _SZ, _SZ, _P, _P, _SZ, _SZ, _SZ, _SZ, _U64,
                                               _U64, _D, C.c_int, _D, _D, C.c_int, C.c_int,
                                               _P]),
    "orc_expert_row_f32": (None, [_P, _SZ, _P, _P, _SZ, _P, _P]),
    "orc_dense_branch_f32": (C.c_int, [_P, _P, _SZ, _SZ, _P, _P, _SZ, _P]),
    "orc_scmoe_layer_f32": (C.c_int, [_P, _P, _P, _SZ, _SZ, _P, _SZ, _SZ, _SZ, _SZ, _D, _P, _P,
                                      _P, _SZ, _D, _D, C.c_int, _P, _P, _P, _P]),
    "orc_simulate_bias_control_f32": (C.c_int, [_P, _SZ, _SZ, _SZ, _SZ, _SZ, _P, _D, _P, _U64,
                                                _SZ, _SZ, _P, _P]),
    "orc_mla_forward_f32": (C.c_int, [_SZ] * 6 + [_D, C.c_int, _P, _P, _SZ, _SZ, _P]),
    "orc_mla_infer_f32": (C.c_int, [_SZ] * 6 + [_D, C.c_int, _P, _P, _SZ, _P, _P, _P]),
}

_REF_PROTOS = {
    "ref_hash2": (_U64, [_U64, _U64]),
    "ref_stream_seed": (_U64, [_U64, _U64]),
    "ref_normal_at": (_D, [_U64, _U64]),
    "ref_seeded_init_f32": (C.c_int, [_U64, _U64, C.c_int, _D, _P]),
    "ref_seeded_init_f64": (C.c_int, [_U64, _U64, C.c_int, _D, _P]),
    "ref_mm_f32": (C.c_int, [_P, _P, _P, _SZ, _SZ, _SZ]),
    "ref_softmax_rows_f32": (C.c_int, [_P, _P, _SZ, _SZ]),
    "ref_expf": (C.c_float, [C.c_float]),
    "ref_route_topk_f32": (C.c_int, [_P, _SZ, _SZ, _P, _SZ, _SZ, _SZ, _SZ, _D, _P, _P, _P, _P, _P,
                                     C.c_int]),
    "ref_route_topk_f64": (C.c_int, [_P, _SZ, _SZ, _P, _SZ, _SZ, _SZ, _SZ, _D, _P, _P, _P, _P, _P,
                                     C.c_int]),
    "ref_route_from_probs_f32": (C.c_int, [_P, _SZ, _SZ, _SZ, _SZ, _SZ, _D, _P, _P, _P, _P]),
    "ref_route_from_probs_f64": (C.c_int, [_P, _SZ, _SZ, _SZ, _SZ, _SZ, _D, _P, _P, _P, _P]),
    "ref_bias_update": (C.c_int, [_SZ, _SZ, _SZ, _SZ, _P, _D, _P, _P, _P, _P]),
    "ref_accumulate_counters": (C.c_int, [_P, _SZ, _SZ, _SZ, _SZ, _P, _P]),
    "ref_routing_stats": (C.c_int, [_P, _P, _SZ, _SZ, _SZ, _SZ, _SZ, _SZ, _P, _P, _P, _P]),
    "ref_moe_forward_f32": (C.c_int, [_P, _SZ, _SZ, _P, _P, _SZ, _SZ, _SZ, _P, _P, _SZ, _SZ,
                                      C.c_int, _P, C.c_int]),
    "ref_moe_forward_f64": (C.c_int, [_P, _SZ, _SZ, _P, _P, _SZ, _SZ, _SZ, _P, _P, _SZ, _SZ,
                                      C.c_int, _P, C.c_int]),
    "ref_rmsnorm_f32": (C.c_int, [_P, _P, _SZ, _SZ, _P]),
    "ref_simulate_bias_control_f32": (C.c_int, [_P, _SZ, _SZ, _SZ, _SZ, _SZ, _P, _D, _P, _U64,
                                                _SZ, _SZ, _P, _P]),
    "ref_mla_forward_f32": (C.c_int, [_SZ] * 6 + [_D, C.c_int, _P, _P, _SZ, _SZ, _P, C.c_int]),
    "ref_mla_infer_f32": (C.c_int, [_SZ] * 6 + [_D, C.c_int, _P, _P, _SZ, _P, _P, _P]),
    "ref_mla_infer_position_check": (C.c_int, [_SZ, _SZ]),
}

_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        build_oracle()
        _orc = _load(ORC_PATH, _ORC_PROTOS)
    return _orc


def ref_available() -> bool:
    if os.path.exists("/root/reference"):
        build_oracle()
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        build_oracle()
        _ref = _load(REF_PATH, _REF_PROTOS)
    return _ref


def ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def ptr_array(arrs):
    """float* const* from a list of numpy arrays (None -> NULL)."""
    arr = (_P * len(arrs))()
    for i, a in enumerate(arrs):
        arr[i] = None if a is None else a.ctypes.data
    return arr


# ---- synthetic recipe ---------------------------------------
def normal_f32(seed: int, n: int, first: int = 0) -> np.ndarray:
    out = np.empty(n, np.float32)
    orc().orc_fill_normal_f32(seed, first, n, ptr(out))
    return out


def normal_f64(seed: int, n: int, first: int = 0) -> np.ndarray:
    out = np.empty(n, np.float64)
    orc().orc_fill_normal_f64(seed, first, n, ptr(out))
    return out


def uniform_f32(seed: int, n: int, variance: float, first: int = 0) -> np.ndarray:
    out = np.empty(n, np.float32)
    rc = orc().orc_seeded_uniform_f32(seed, first, n, variance, ptr(out))
    assert rc == 0
    return out


def stream_seed(seed: int, sid: int) -> int:
    return int(orc().orc_stream_seed(seed, sid))


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round fp32 to bf16 (RNE) and widen back to fp32."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


# ---- oracle calls -----------------------------------------------------------
def orc_route_topk(x, w, n_ffn, n_zero, k, ke, mu=0.0, bias=None, want_probs=False):
    x = np.ascontiguousarray(x, np.float32)
    w = np.ascontiguousarray(w, np.float32)
    T, d = x.shape
    E = n_ffn + n_zero
    b = np.zeros(E) if bias is None else np.ascontiguousarray(bias, np.float64)
    idx = np.empty(T * k, np.uint32)
    g = np.empty(T * k, np.float64)
    c = np.empty(T, np.uint32)
    probs = np.empty((T, E), np.float32) if want_probs else None
    rc = orc().orc_route_topk_f32(ptr(x), T, d, ptr(w), n_ffn, n_zero, k, ke, mu, ptr(b),
                                  ptr(idx), ptr(g), ptr(c), ptr(probs))
    return rc, idx, g, c, probs


def orc_route_topk_f64(x, w, n_ffn, n_zero, k, ke, mu=0.0, bias=None):
    """RouterState<double> route_topk restated (libm exp)."""
    x = np.ascontiguousarray(x, np.float64)
    w = np.ascontiguousarray(w, np.float64)
    T, d = x.shape
    E = n_ffn + n_zero
    b = np.zeros(E) if bias is None else np.ascontiguousarray(bias, np.float64)
    idx = np.empty(T * k, np.uint32)
    g = np.empty(T * k, np.float64)
    c = np.empty(T, np.uint32)
    probs = np.empty((T, E), np.float64)
    rc = orc().orc_route_topk_f64(ptr(x), T, d, ptr(w), n_ffn, n_zero, k, ke, mu, ptr(b),
                                  ptr(idx), ptr(g), ptr(c), ptr(probs))
    return rc, idx, g, c, probs


def orc_moe_forward(x, idx, gates, k, n_ffn, n_zero, w_in, w_out, gamma_ffn=1.0,
                    gamma_zero=1.0, renorm=False):
    x = np.ascontiguousarray(x, np.float32)
    T, d = x.shape
    I = next(w for w in w_in if w is not None).shape[1]
    out = np.empty((T, d), np.float32)
    w_in = [None if w is None else np.ascontiguousarray(w, np.float32) for w in w_in]
    w_out = [None if w is None else np.ascontiguousarray(w, np.float32) for w in w_out]
    rc = orc().orc_moe_forward_f32(ptr(x), T, d, ptr(np.ascontiguousarray(idx, np.uint32)),
                                   ptr(np.ascontiguousarray(gates, np.float64)), k, n_ffn, n_zero,
                                   ptr_array(w_in), ptr_array(w_out), I, gamma_ffn, gamma_zero,
                                   int(renorm), ptr(out))
    return rc, out


def orc_moe_forward_streamed(x, idx, gates, k, n_ffn, n_zero, inter, seed, stream0=100,
                             bf16=True, gamma_ffn=1.0, gamma_zero=1.0, renorm=False,
                             threads=None):
    """moe_forward on a token sample with the expert bank regenerated per
    expert from its seeded_init Uniform streams (variance 1/d), bf16-rounded
    as the device bank stores them (configs B/C; oracle/scmoe_oracle.c)."""
    x = np.ascontiguousarray(x, np.float32)
    T, d = x.shape
    out = np.empty((T, d), np.float32)
    rc = orc().orc_moe_forward_streamed_f32(
        ptr(x), T, d, ptr(np.ascontiguousarray(idx, np.uint32)),
        ptr(np.ascontiguousarray(gates, np.float64)), k, n_ffn, n_zero, inter, seed, stream0,
        1.0 / d, int(bf16), gamma_ffn, gamma_zero, int(renorm), threads or os.cpu_count() or 1,
        ptr(out))
    return rc, out


def routing_stats(fn, idx, cnt, k, n, z, ke, groups):
    """fn: orc().orc_routing_stats or ref().ref_routing_stats -> (rc, mean, std, load, lb)."""
    idx = np.ascontiguousarray(idx, np.uint32)
    cnt = np.ascontiguousarray(cnt, np.uint32)
    mean, std = C.c_double(), C.c_double()
    load = np.empty(n + z)
    lb = np.empty(groups + (1 if z else 0)) if groups else None
    rc = fn(ptr(idx), ptr(cnt), len(cnt), k, n, z, ke, groups, C.byref(mean), C.byref(std),
            ptr(load), ptr(lb))
    return rc, mean.value, std.value, load, lb


def random_decision(seed, T, k, n, z):
    """Indices with distinct experts per token, ffn_count consistent with them."""
    rng = np.random.default_rng(seed)
    rows = [rng.choice(n + z, k, replace=False) for _ in range(T)]
    idx = (np.stack(rows) if rows else np.zeros((0, k))).astype(np.uint32)
    return idx.ravel(), (idx < n).sum(1).astype(np.uint32)


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ---- MLA (blocks.hpp:38-181) ---------------------------------------------------
MLA_NAMES = ("w_dq", "w_uq", "w_qr", "w_dkv", "w_uk", "w_uv", "w_kr", "w_o")


def mla_shapes(d, dq, dkv, H, dhc, dhr):
    return [(d, dq), (dq, H * dhc), (dq, H * dhr), (d, dkv), (dkv, H * dhc), (dkv, H * dhc),
            (d, dhr), (H * dhc, d)]


def mla_weights(d, dq, dkv, H, dhc, dhr, seed=3):
    """MlaFixture-like weights (tests/test_blocks.cpp:27-66) with the Uniform
    device-reproducible init of variance 1/d_model, stream ids 0..7."""
    return [uniform_f32(stream_seed(seed, i), r * c, 1.0 / d).reshape(r, c)
            for i, (r, c) in enumerate(mla_shapes(d, dq, dkv, H, dhc, dhr))]


def mla_forward(lib, dims, w, h, seq_len, base=1.0e4, va=1, threads=1):
    d, dq, dkv, H, dhc, dhr = dims
    h = np.ascontiguousarray(h, np.float32)
    rows = h.shape[0]
    out = np.zeros((rows, d), np.float32)
    ws = [np.ascontiguousarray(x, np.float32) for x in w]
    args = [d, dq, dkv, H, dhc, dhr, base, va, ptr_array(ws), ptr(h), rows, seq_len, ptr(out)]
    if lib is _ref:
        args.append(threads)
    rc = (lib.ref_mla_forward_f32 if lib is _ref else lib.orc_mla_forward_f32)(*args)
    return rc, out


def mla_infer(lib, dims, w, h, base=1.0e4, va=1):
    d, dq, dkv, H, dhc, dhr = dims
    h = np.ascontiguousarray(h, np.float32)
    T = h.shape[0]
    out = np.zeros((T, d), np.float32)
    ckv = np.zeros((T, dkv), np.float32)
    kr = np.zeros((T, dhr), np.float32)
    ws = [np.ascontiguousarray(x, np.float32) for x in w]
    fn = lib.ref_mla_infer_f32 if lib is _ref else lib.orc_mla_infer_f32
    rc = fn(d, dq, dkv, H, dhc, dhr, base, va, ptr_array(ws), ptr(h), T, ptr(out), ptr(ckv),
            ptr(kr))
    return rc, out, ckv, kr
