"""Multi-head latent attention, forward value.

Mirrors the reference's MLA API (blocks.hpp:19-181) over the C ABI
(include/scmoe.h, scmoe_mla_*):

* ``mla_scale_factors(d_model, d_q, d_kv)``      -- blocks.hpp:19-26
* ``MlaParams``  (weights + dims, device-resident) -- blocks.hpp:38-58
* ``mla_block(h, params, seq_len)``               -- blocks.hpp:73-102 (value)
* ``MlaCache`` + ``mla_infer_step(params, cache, h_t, position)`` -- :106-181

All arithmetic runs in the CUDA kernels of csrc/mla.cu, bitwise equal to the
reference's fp32 path; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Optional, Sequence

import numpy as np

from . import Context, ParameterError, _P, _SZ, _ptr, default_context, lib

WEIGHT_NAMES = ("w_dq", "w_uq", "w_qr", "w_dkv", "w_uk", "w_uv", "w_kr", "w_o")


def mla_scale_factors(d_model: int, d_q: int, d_kv: int):
    """blocks.hpp:19-26."""
    if d_model == 0 or d_q == 0 or d_kv == 0:
        raise ParameterError("mla_scale_factors: dims must be positive")
    return math.sqrt(d_model / d_q), math.sqrt(d_model / d_kv)


class MlaParams:
    """MlaParams<float>: dims, rope base, variance alignment and the eight
    projection matrices (row-major, shapes as in blocks.hpp:44-51).  Weights are
    uploaded once per context (device residency); ``invalidate()`` after
    changing them."""

    def __init__(self, d_model: int, d_q: int, d_kv: int, n_heads: int, d_head_c: int,
                 d_head_r: int, weights: Sequence, rope_base: float = 1.0e6,
                 variance_alignment: bool = True, precision: int = 0):
        self.d_model, self.d_q, self.d_kv = d_model, d_q, d_kv
        self.n_heads, self.d_head_c, self.d_head_r = n_heads, d_head_c, d_head_r
        self.rope_base, self.variance_alignment = rope_base, variance_alignment
        if isinstance(weights, dict):
            weights = [weights[n] for n in WEIGHT_NAMES]
        self.weights = list(weights)  # numpy arrays or CUDA torch tensors
        # 0 = SCMOE_PREC_F32_EXACT (bitwise), 1 = SCMOE_PREC_BF16 (tensor cores)
        self.precision = precision
        self._dev = None

    def shapes(self):
        d, dq, dkv, H, c, r = (self.d_model, self.d_q, self.d_kv, self.n_heads, self.d_head_c,
                               self.d_head_r)
        return [(d, dq), (dq, H * c), (dq, H * r), (d, dkv), (dkv, H * c), (dkv, H * c), (d, r),
                (H * c, d)]

    def alpha_q(self) -> float:
        return mla_scale_factors(self.d_model, self.d_q, self.d_kv)[0] \
            if self.variance_alignment else 1.0

    def alpha_kv(self) -> float:
        return mla_scale_factors(self.d_model, self.d_q, self.d_kv)[1] \
            if self.variance_alignment else 1.0

    def invalidate(self):
        """Drop the device copy (the next call re-uploads the weights)."""
        if self._dev is not None:
            try:
                lib().scmoe_mla_destroy(self._dev[0].handle, self._dev[1])
            finally:
                self._dev = None

    def device(self, ctx: Context):
        if self._dev is not None and self._dev[0] is ctx:
            h, prec = self._dev[1], self._dev[2]
            if prec != self.precision:  # precision switched after the upload
                ctx._check(lib().scmoe_mla_set_precision(ctx.handle, h, int(self.precision)))
                self._dev = (ctx, h, self.precision)
            return h
        self.invalidate()  # another context's copy
        h = _P()
        ctx._check(lib().scmoe_mla_create(ctx.handle, self.d_model, self.d_q, self.d_kv,
                                          self.n_heads, self.d_head_c, self.d_head_r,
                                          self.rope_base, int(self.variance_alignment),
                                          C.byref(h)))
        try:  # the handle is destroyed if any weight or the precision is rejected
            for i, (w, shp) in enumerate(zip(self.weights, self.shapes())):
                if tuple(w.shape) != shp:
                    raise ParameterError(f"mla: {WEIGHT_NAMES[i]} has shape {tuple(w.shape)}, "
                                         f"expected {shp}")
                if hasattr(w, "data_ptr"):  # CUDA tensor
                    ctx._check(lib().scmoe_mla_set_weight(ctx.handle, h, i,
                                                          w.contiguous().data_ptr()))
                else:
                    a = np.ascontiguousarray(w, np.float32)
                    ctx._check(lib().scmoe_mla_set_weight_host(ctx.handle, h, i, _ptr(a)))
            if self.precision:
                ctx._check(lib().scmoe_mla_set_precision(ctx.handle, h, int(self.precision)))
        except Exception:
            lib().scmoe_mla_destroy(ctx.handle, h)
            raise
        self._dev = (ctx, h, self.precision)
        return h

    def __del__(self):
        try:
            if self._dev is not None:
                lib().scmoe_mla_destroy(self._dev[0].handle, self._dev[1])
        except Exception:
            pass


def mla_block(h, p: MlaParams, seq_len: int, ctx: Optional[Context] = None,
              out=None):
    """Value of mla_block (blocks.hpp:73-102) over packed sequences of
    ``seq_len`` rows.  ``h``: numpy [rows, d] (host API) or a CUDA fp32 tensor
    (device API, stream-ordered on the context's stream)."""
    ctx = ctx or default_context()
    m = p.device(ctx)
    if hasattr(h, "data_ptr"):
        import torch
        rows = h.shape[0]
        out = torch.empty((rows, p.d_model), dtype=torch.float32, device=h.device) \
            if out is None else out
        ctx._check(lib().scmoe_mla_forward(ctx.handle, m, h.contiguous().data_ptr(), rows,
                                           seq_len, out.data_ptr()))
        return out
    h = np.ascontiguousarray(h, np.float32)
    rows = h.shape[0]
    out = np.empty((rows, p.d_model), np.float32)
    ctx._check(lib().scmoe_mla_forward_host(ctx.handle, m, _ptr(h), rows, seq_len, _ptr(out)))
    return out


class MlaCache:
    """MlaCache (blocks.hpp:106-112): the compressed KV stream (c_kv, rotated
    k_r), device-resident, plus the expanded content keys / values of the
    cached rows (row-wise, so bitwise the reference's re-expansion)."""

    def __init__(self, p: MlaParams, capacity_hint: int = 256, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.p = p
        self._h = _P()
        self.ctx._check(lib().scmoe_mla_cache_create(self.ctx.handle, p.device(self.ctx),
                                                     capacity_hint, C.byref(self._h)))

    def length(self) -> int:
        n = _SZ()
        self.ctx._check(lib().scmoe_mla_cache_length(self.ctx.handle, self._h, C.byref(n)))
        return int(n.value)

    def read(self):
        """(c_kv [n, d_kv], k_r [n, d_head_r]) as numpy."""
        n = self.length()
        ckv = np.empty((n, self.p.d_kv), np.float32)
        kr = np.empty((n, self.p.d_head_r), np.float32)
        self.ctx._check(lib().scmoe_mla_cache_read_host(self.ctx.handle,
                                                        self.p.device(self.ctx), self._h,
                                                        _ptr(ckv), _ptr(kr)))
        return ckv, kr

    def __del__(self):
        try:
            lib().scmoe_mla_cache_destroy(self.ctx.handle, self._h)
        except Exception:
            pass


def mla_infer_step(p: MlaParams, cache: MlaCache, h_t, position: int, out=None):
    """One decode step (blocks.hpp:129-181): h_t [1, d] at ``position``; the
    cache must hold exactly ``position`` rows (StateError otherwise)."""
    ctx = cache.ctx
    m = p.device(ctx)
    if hasattr(h_t, "data_ptr"):
        import torch
        out = torch.empty((1, p.d_model), dtype=torch.float32, device=h_t.device) \
            if out is None else out
        ctx._check(lib().scmoe_mla_infer_step(ctx.handle, m, cache._h,
                                              h_t.contiguous().data_ptr(), position,
                                              out.data_ptr()))
        return out
    h_t = np.ascontiguousarray(h_t, np.float32).reshape(1, p.d_model)
    out = np.empty((1, p.d_model), np.float32)
    ctx._check(lib().scmoe_mla_infer_step_host(ctx.handle, m, cache._h, _ptr(h_t), position,
                                               _ptr(out)))
    return out


class ScMoELayer:
    """The full ScMoE layer of Model::build_layer (model.hpp:355-409), forward
    value: two MLA blocks, the dense shortcut FFN and the MoE branch with
    zero-computation experts, wired as the reference wires them (scmoe: the
    MoE reads rmsnorm(a1), so it can run beside dense FFN + MLA2).

    ``mla1``/``mla2``: MlaParams; ``dense``: layer.DenseFFN; ``router``:
    RouterState; ``bank``: ExpertBank (PREC_BF16 for the tcgen05 path);
    norms: gain vectors [d] (numpy)."""

    def __init__(self, mla1: MlaParams, mla2: MlaParams, dense, router, bank, norm1, norm_ffn,
                 norm2, norm_moe, ctx: Optional[Context] = None):
        import torch
        self.ctx = ctx or default_context()
        self.mla1, self.mla2, self.dense, self.router, self.bank = mla1, mla2, dense, router, bank
        self.d = mla1.d_model
        self.norms = [torch.from_numpy(np.ascontiguousarray(g, np.float32)).cuda()
                      for g in (norm1, norm_ffn, norm2, norm_moe)]

    def forward(self, x, seq_len: int, renormalize: bool = False, overlap: bool = True,
                want_intermediates: bool = False):
        """x: CUDA fp32 tensor [T, d] (device API) or numpy (copied in/out).
        Returns (out, indices, gates, ffn_count[, a1, a3])."""
        import torch
        host = not hasattr(x, "data_ptr")
        xt = torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda() if host else x
        T = xt.shape[0]
        K = self.router.top_k
        dev = xt.device
        out = torch.empty((T, self.d), dtype=torch.float32, device=dev)
        idx = torch.empty(T * K, dtype=torch.int32, device=dev)
        gates = torch.empty(T * K, dtype=torch.float64, device=dev)
        cnt = torch.empty(T, dtype=torch.int32, device=dev)
        a1 = torch.empty_like(out) if want_intermediates else None
        a3 = torch.empty_like(out) if want_intermediates else None
        c = self.ctx
        c._check(lib().scmoe_layer_full_forward(
            c.handle, self.mla1.device(c), self.mla2.device(c), self.dense.bank,
            self.router.device(c), self.bank.device(c), *[g.data_ptr() for g in self.norms],
            xt.contiguous().data_ptr(), T, seq_len, int(renormalize), int(overlap),
            idx.data_ptr(), gates.data_ptr(), cnt.data_ptr(),
            None if a1 is None else a1.data_ptr(), None if a3 is None else a3.data_ptr(),
            out.data_ptr()))
        res = [out, idx, gates, cnt] + ([a1, a3] if want_intermediates else [])
        if host:
            c.synchronize()
            res = [t.cpu().numpy() for t in res]
            res[1] = res[1].view(np.uint32)
            res[3] = res[3].view(np.uint32)
        return tuple(res)
