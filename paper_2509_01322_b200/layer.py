"""Device-tier ScMoE layer: router + expert bank resident in HBM, inputs and
outputs as device pointers (e.g. torch CUDA tensors' data_ptr()).

This is the serving/benchmark entry point; the reference-shaped API in
``paper_2509_01322_b200`` (route_topk, moe_forward, ...) is the host tier.
Synthetic weights follow SURVEY.md 8(d): router W_r = seeded_init Uniform
(variance 1/d) of CounterRng(seed).stream(0); expert e's w_in / w_out =
seeded_init Uniform of stream(100 + 2e) / stream(101 + 2e), generated on the
device bit-for-bit as the reference's rng.hpp would on the host.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

from . import (PREC_BF16, Context, GammaMode, _P, lib)


@dataclass
class LayerShape:
    d: int = 6144
    n_ffn: int = 512
    n_zero: int = 256
    top_k: int = 12
    k_expected: int = 8
    inter: int = 2048
    m: int = 1
    gamma_mode: int = int(GammaMode.FfnOnly)
    precision: int = PREC_BF16

    @property
    def E(self) -> int:
        return self.n_ffn + self.n_zero


LONGCAT = LayerShape()
TINY = LayerShape(d=256, n_ffn=8, n_zero=4, top_k=2, k_expected=1, inter=128, precision=0)


class DeviceLayer:
    def __init__(self, ctx: Context, shape: LayerShape, seed: int = 5, mu: float = 0.0,
                 mu_decay: float = 1.0):
        self.ctx, self.shape, self.seed = ctx, shape, seed
        L = lib()
        s = shape
        self.router = _P()
        ctx._check(L.scmoe_router_create(ctx.handle, s.d, s.n_ffn, s.n_zero, s.top_k,
                                         s.k_expected, mu, mu_decay, C.byref(self.router)))
        # router weights: generated on the device into a scratch buffer
        wbuf = _P()
        nbytes = s.d * s.E * 4
        ctx._check(L.scmoe_device_alloc(ctx.handle, nbytes, C.byref(wbuf)))
        sd = int(L.scmoe_rng_stream_seed(seed, 0))
        ctx._check(L.scmoe_rng_fill_uniform(ctx.handle, sd, 0, s.d * s.E, 1.0 / s.d, wbuf))
        ctx._check(L.scmoe_router_set_weights(ctx.handle, self.router, wbuf))
        ctx.synchronize()
        ctx._check(L.scmoe_device_free(ctx.handle, wbuf))
        self.bank = _P()
        ctx._check(L.scmoe_bank_create(ctx.handle, s.n_ffn, s.d, s.inter, s.precision, s.m,
                                       s.gamma_mode, C.byref(self.bank)))
        ctx._check(L.scmoe_bank_init_uniform(ctx.handle, self.bank, seed, 100, 1.0 / s.d))

    def bank_bytes(self) -> int:
        return int(lib().scmoe_bank_device_bytes(self.bank))

    def forward(self, a1: int, a3: int, gain: Optional[int], tokens: int, idx: int, gates: int,
                ffn_count: int, out: int, renormalize: bool = False):
        """Device pointers; stream-ordered on the context's stream."""
        self.ctx._check(lib().scmoe_layer_forward(self.ctx.handle, self.router, self.bank, a1, a3,
                                                  gain, tokens, int(renormalize), idx, gates,
                                                  ffn_count, out))

    # ---- PID controller (router.hpp:144-176, model.hpp:235-244) ------------
    def accumulate(self, idx: int, tokens: int):
        """accumulate_counters on the device (indices as a device pointer)."""
        self.ctx._check(lib().scmoe_accumulate_counters(self.ctx.handle, self.router, idx, tokens))

    def bias_update(self, want_delta: bool = True):
        """bias_update; returns the applied deltas (numpy) when want_delta."""
        import numpy as np
        delta = np.empty(self.shape.E, np.float64) if want_delta else None
        self.ctx._check(lib().scmoe_bias_update(self.ctx.handle, self.router,
                                                None if delta is None else
                                                delta.ctypes.data_as(_P)))
        return delta

    def tokens_seen(self) -> int:
        seen = C.c_uint64()
        self.ctx._check(lib().scmoe_router_get_counters_host(self.ctx.handle, self.router, None,
                                                             C.byref(seen)))
        return int(seen.value)

    def bias(self):
        import numpy as np
        b = np.empty(self.shape.E, np.float64)
        self.ctx._check(lib().scmoe_router_get_bias_host(self.ctx.handle, self.router,
                                                         b.ctypes.data_as(_P)))
        return b

    def counters(self):
        import numpy as np
        r = np.empty(self.shape.E, np.uint64)
        seen = C.c_uint64()
        self.ctx._check(lib().scmoe_router_get_counters_host(self.ctx.handle, self.router,
                                                             r.ctypes.data_as(_P), C.byref(seen)))
        return r, int(seen.value)

    def router_weights(self):
        """The router projection [d, E] (host copy), e.g. for an oracle check."""
        import numpy as np
        s = self.shape
        w = np.empty(s.d * s.E, np.float32)
        L = lib()
        sd = int(L.scmoe_rng_stream_seed(self.seed, 0))
        dev = _P()
        self.ctx._check(L.scmoe_device_alloc(self.ctx.handle, w.nbytes, C.byref(dev)))
        self.ctx._check(L.scmoe_rng_fill_uniform(self.ctx.handle, sd, 0, w.size, 1.0 / s.d, dev))
        self.ctx._check(L.scmoe_copy_d2h(self.ctx.handle, w.ctypes.data_as(_P), dev, w.nbytes))
        L.scmoe_device_free(self.ctx.handle, dev)
        return w.reshape(s.d, s.E)

    def forward_batches(self, a1s, a3s, gain: Optional[int], tokens: int, idxs, gatess, cnts,
                        outs, renormalize: bool = False):
        """Pipelined micro-batches (scmoe_layer_forward_batches): lists of device
        pointers, one per batch.  Buffers of consecutive batches must not alias."""
        n = len(a1s)
        arr = lambda xs: (C.c_void_p * n)(*xs)  # noqa: E731
        self.ctx._check(lib().scmoe_layer_forward_batches(
            self.ctx.handle, self.router, self.bank, n, arr(a1s),
            arr(a3s) if a3s is not None else None, gain, tokens, int(renormalize), arr(idxs),
            arr(gatess), arr(cnts), arr(outs)))

    def forward_host(self, a1, a3, gain, tokens: int, idx, gates, ffn_count, out,
                     renormalize: bool = False):
        """Host (ideally pinned) numpy buffers; copies in, runs, copies out."""
        p = lambda a: None if a is None else a.ctypes.data_as(_P)  # noqa: E731
        self.ctx._check(lib().scmoe_layer_forward_host(self.ctx.handle, self.router, self.bank,
                                                       p(a1), p(a3), p(gain), tokens,
                                                       int(renormalize), p(idx), p(gates),
                                                       p(ffn_count), p(out)))

    def routing_stats(self, idx: int, ffn_count: int, tokens: int, lb_groups: int = 0) -> dict:
        """Routing statistics of a forward's routing outputs (device pointers):
        mean/std activated FFN experts, per-expert load, LB group frequencies
        (scmoe_routing_stats)."""
        import numpy as np
        s = self.shape
        mean, std = C.c_double(), C.c_double()
        load = np.empty(s.E, np.float64)
        lb = np.empty(lb_groups + (1 if s.n_zero else 0)) if lb_groups else None
        self.ctx._check(lib().scmoe_routing_stats(
            self.ctx.handle, idx, ffn_count, tokens, s.top_k, s.n_ffn, s.n_zero, s.k_expected,
            lb_groups, C.byref(mean), C.byref(std), load.ctypes.data_as(_P),
            None if lb is None else lb.ctypes.data_as(_P)))
        out = {"mean_activated_ffn": mean.value, "std_activated_ffn": std.value,
               "per_expert_load": load}
        if lb is not None:
            out["lb_group_frequencies"] = lb
        return out

    def forward_host_batches(self, a1s, a3s, gain, tokens: int, idxs, gatess, cnts, outs,
                             renormalize: bool = False):
        """A stream of host batches (scmoe_layer_forward_host_batches): lists of
        (ideally pinned) numpy arrays, one per batch; input copies, compute and
        output copies of neighbouring batches overlap.  idxs/gatess/cnts may be
        None."""
        n = len(a1s)
        p = lambda a: None if a is None else a.ctypes.data_as(_P)  # noqa: E731
        arr = lambda xs: None if xs is None else (C.c_void_p * n)(  # noqa: E731
            *[None if x is None else x.ctypes.data for x in xs])
        self.ctx._check(lib().scmoe_layer_forward_host_batches(
            self.ctx.handle, self.router, self.bank, n, arr(a1s), arr(a3s), p(gain), tokens,
            int(renormalize), arr(idxs), arr(gatess), arr(cnts), arr(outs)))

    def close(self):
        """Free the device router and bank (also done when the object dies
        while its context is still open)."""
        L = lib()
        if not self.ctx.handle:  # closed context: its handles can no longer be used
            self.bank = self.router = _P()
            return
        if self.bank:
            L.scmoe_bank_destroy(self.ctx.handle, self.bank)
            self.bank = _P()
        if self.router:
            L.scmoe_router_destroy(self.ctx.handle, self.router)
            self.router = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DenseFFN:
    """Dense shortcut-path FFN of the ScMoE layer (model.hpp:390-391,
    blocks.hpp:397-402): out = a1 + silu(rmsnorm(a1, gain) W_in) W_out, bf16 weights
    on the tcgen05 grouped GEMM (a one-expert bank).  Weights: seeded_init
    Uniform(1/d) on the device (streams stream0, stream0 + 1), or set from host
    fp32 arrays w_in [d, inter], w_out [inter, d]."""

    def __init__(self, ctx: Context, d: int, inter: int, seed: int = 9, stream0: int = 7000,
                 w_in=None, w_out=None):
        self.ctx, self.d, self.inter = ctx, d, inter
        L = lib()
        self.bank = _P()
        ctx._check(L.scmoe_bank_create(ctx.handle, 1, d, inter, PREC_BF16, 1,
                                       int(GammaMode.Off), C.byref(self.bank)))
        try:
            if w_in is not None:
                import numpy as np
                wi = np.ascontiguousarray(w_in, np.float32)
                wo = np.ascontiguousarray(w_out, np.float32)
                ctx._check(L.scmoe_bank_set_expert_host(ctx.handle, self.bank, 0,
                                                        wi.ctypes.data_as(_P),
                                                        wo.ctypes.data_as(_P)))
            else:
                ctx._check(L.scmoe_bank_init_uniform(ctx.handle, self.bank, seed, stream0,
                                                     1.0 / d))
        except Exception:
            self.close()
            raise

    def forward(self, a1: int, gain: Optional[int], tokens: int, out: int,
                ctx: Optional[Context] = None):
        """Device pointers; stream-ordered on ctx's stream (default: the owner's)."""
        c = ctx or self.ctx
        c._check(lib().scmoe_dense_ffn(c.handle, self.bank, a1, gain, tokens, out))

    def close(self):
        if self.bank and self.ctx.handle:
            lib().scmoe_bank_destroy(self.ctx.handle, self.bank)
        self.bank = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
