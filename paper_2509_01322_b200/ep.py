"""Expert-parallel ScMoE layer over the GPUs of one node: a
thin caller of the device-resident C-ABI orchestration (scmoe_ep_*,
csrc/ep.cu).

Router and bias replicated, tokens sharded, FFN experts block-partitioned
(rank g owns [g*N/G, (g+1)*N/G)), zero experts local.  Every
layer call runs on the device without host synchronisation: routing, the
dispatch plan, an on-device exchange of the slot-count matrix, peer stores
of the bf16 rows over NVLink, grouped GEMMs whose GEMM2 epilogue returns the
rows to their source rank, and the rank-order combine (blocks.hpp:251-274).
The output is bitwise equal to the single-GPU layer.  torch.distributed is
only used here to hand rank 0's NCCL unique id to the other ranks (a C++
host would use its own launcher); torch streams/tensors are interop.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np
import torch

from . import PREC_BF16, Context, GammaMode, _P, lib
from .layer import LayerShape


def unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 creates it, every rank passes it)."""
    n = int(lib().scmoe_ep_unique_id_bytes())
    buf = (C.c_char * n)()
    rc = lib().scmoe_ep_unique_id(buf)
    if rc != 0:
        raise RuntimeError(f"scmoe_ep_unique_id failed ({rc})")
    return bytes(buf)


def broadcast_unique_id(group=None) -> bytes:
    """rank 0's unique id on every rank of `group` (torch.distributed plumbing)."""
    import torch.distributed as dist
    obj = [unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                               group=group)
    return obj[0]


class ExpertParallelLayer:
    """One ScMoE MoE branch sharded over `world` ranks (one GPU each).

    Synthetic weights as the single-GPU DeviceLayer(seed): router W_r =
    seeded_init Uniform of CounterRng(seed).stream(0); this rank's experts =
    global experts [rank*N/G, (rank+1)*N/G) from streams 100 + 2e / 101 + 2e."""

    def __init__(self, ctx: Context, shape: LayerShape, rank: int, world: int, seed: int,
                 uid: bytes, max_tokens: int, max_recv_rows: int = 0, mu: float = 0.0,
                 mu_decay: float = 1.0):
        if shape.precision != PREC_BF16:
            raise ValueError("expert parallelism runs the bf16 tensor-core bank")
        if shape.n_ffn % world:
            raise ValueError("world size must divide the FFN expert count")
        self.ctx, self.shape, self.rank, self.world = ctx, shape, rank, world
        self.n_local = shape.n_ffn // world
        self.first = rank * self.n_local
        self.max_tokens = max_tokens
        self.stream = torch.cuda.Stream()
        ctx.set_stream(self.stream.cuda_stream)
        L = lib()
        s = shape
        self.router = _P()
        ctx._check(L.scmoe_router_create(ctx.handle, s.d, s.n_ffn, s.n_zero, s.top_k,
                                         s.k_expected, mu, mu_decay, C.byref(self.router)))
        w = torch.empty(s.d * s.E, dtype=torch.float32, device="cuda")
        ctx._check(L.scmoe_rng_fill_uniform(ctx.handle, int(L.scmoe_rng_stream_seed(seed, 0)), 0,
                                            s.d * s.E, 1.0 / s.d, w.data_ptr()))
        ctx._check(L.scmoe_router_set_weights(ctx.handle, self.router, w.data_ptr()))
        self.bank = _P()
        ctx._check(L.scmoe_bank_create(ctx.handle, self.n_local, s.d, s.inter, s.precision, s.m,
                                       s.gamma_mode, C.byref(self.bank)))
        ctx._check(L.scmoe_bank_init_uniform_shard(ctx.handle, self.bank, seed, 100, 1.0 / s.d,
                                                   self.first))
        ctx.synchronize()
        self.dense_bank = None
        self.ep = _P()
        uid_buf = C.create_string_buffer(uid, len(uid))
        ctx._check(L.scmoe_ep_create(ctx.handle, world, rank, uid_buf, s.d, s.n_ffn, s.n_zero,
                                     s.top_k, max_tokens, max_recv_rows, C.byref(self.ep)))

    # -- configuration ---------------------------------------------------------
    def enable_dense(self, inter: int, seed: int, stream0: int = 7000, reserve_sms: int = 16):
        """Dense shortcut FFN dd = a1 + ffn_block(rmsnorm(a1)) (model.hpp:390-391),
        one-expert bf16 bank, run by forward(dense=True) beside the MoE branch."""
        L = lib()
        b = _P()
        self.ctx._check(L.scmoe_bank_create(self.ctx.handle, 1, self.shape.d, inter, PREC_BF16, 1,
                                            int(GammaMode.Off), C.byref(b)))
        self.ctx._check(L.scmoe_bank_init_uniform(self.ctx.handle, b, seed, stream0,
                                                  1.0 / self.shape.d))
        self.ctx.synchronize()
        self.dense_bank = b
        self.ctx._check(L.scmoe_ep_set_dense_reserve(self.ep, reserve_sms))

    def set_comm(self, on: bool):
        """False: row transfers replaced by no-ops (timing reference only)."""
        self.ctx._check(lib().scmoe_ep_set_comm(self.ep, int(on)))

    # -- forward -----------------------------------------------------------------
    def _outputs(self, T: int):
        s = self.shape
        return (torch.empty(T, s.d, dtype=torch.float32, device="cuda"),
                torch.empty(T * s.top_k, dtype=torch.int32, device="cuda"),
                torch.empty(T * s.top_k, dtype=torch.float64, device="cuda"),
                torch.empty(T, dtype=torch.int32, device="cuda"))

    def forward(self, a1: torch.Tensor, a3: Optional[torch.Tensor], gain: Optional[torch.Tensor],
                T: int, renormalize: bool = False, dense: bool = False):
        """(out, idx, gates, ffn_count) of this rank's T tokens; dense=True uses
        the dense branch's dd as the residual (a3 ignored)."""
        if dense and self.dense_bank is None:
            raise ValueError("enable_dense() first")
        cur = torch.cuda.current_stream()
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            out, idx, gates, cnt = self._outputs(T)
            self.ctx._check(lib().scmoe_ep_layer_forward(
                self.ep, self.router, self.bank, self.dense_bank if dense else None, a1.data_ptr(),
                None if (a3 is None or dense) else a3.data_ptr(),
                None if gain is None else gain.data_ptr(), T, int(renormalize), idx.data_ptr(),
                gates.data_ptr(), cnt.data_ptr(), out.data_ptr()))
        cur.wait_stream(self.stream)
        for t in (out, idx, gates, cnt, a1) + ((a3,) if a3 is not None else ()):
            t.record_stream(cur)
        return out, idx, gates, cnt

    def forward_batches(self, a1s: List[torch.Tensor], a3s, gain, T: int,
                        renormalize: bool = False, corun_router: bool = False):
        """A pipelined stream of batches (scmoe_ep_layer_forward_batches);
        returns [(out, idx, gates, ffn_count)] -- identical to forward() calls."""
        n = len(a1s)
        cur = torch.cuda.current_stream()
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            res = [self._outputs(T) for _ in range(n)]
            arr = lambda xs: (C.c_void_p * n)(*xs)  # noqa: E731
            self.ctx._check(lib().scmoe_ep_layer_forward_batches(
                self.ep, self.router, self.bank, n, arr([a.data_ptr() for a in a1s]),
                None if a3s is None else arr([a.data_ptr() for a in a3s]),
                None if gain is None else gain.data_ptr(), T, int(renormalize), int(corun_router),
                arr([r[1].data_ptr() for r in res]), arr([r[2].data_ptr() for r in res]),
                arr([r[3].data_ptr() for r in res]), arr([r[0].data_ptr() for r in res])))
        cur.wait_stream(self.stream)
        for r in res:
            for t in r:
                t.record_stream(cur)
        return res

    def forward_host_batches(self, a1s, a3s, outs, gain, T: int, renormalize: bool = False):
        """Host tier for a stream of batches (pinned host tensors in, `outs`
        filled): copy-in of batch i+1 and copy-out of batch i-1 run on copy
        streams while batch i computes (device inputs double buffered)."""
        cur = torch.cuda.current_stream()
        cin, cout = torch.cuda.Stream(), torch.cuda.Stream()
        n = len(a1s)
        dev = [dict(a1=torch.empty(a1s[0].shape, dtype=a1s[0].dtype, device="cuda"),
                    a3=None if a3s is None else torch.empty(a3s[0].shape, dtype=a3s[0].dtype,
                                                           device="cuda")) for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(n)]
        ev_used = [torch.cuda.Event() for _ in range(n)]
        cin.wait_stream(cur)
        cout.wait_stream(cur)

        def copy_in(i):
            with torch.cuda.stream(cin):
                if i >= 2:
                    cin.wait_event(ev_used[i - 2])
                b = dev[i % 2]
                b["a1"].copy_(a1s[i], non_blocking=True)
                if a3s is not None:
                    b["a3"].copy_(a3s[i], non_blocking=True)
                ev_in[i].record(cin)

        routing = []
        copy_in(0)
        for i in range(n):
            if i + 1 < n:
                copy_in(i + 1)
            cur.wait_event(ev_in[i])
            b = dev[i % 2]
            out, idx, gates, cnt = self.forward(b["a1"], b["a3"], gain, T, renormalize)
            ev_used[i].record(cur)
            with torch.cuda.stream(cout):
                cout.wait_event(ev_used[i])
                outs[i].copy_(out.view(outs[i].shape), non_blocking=True)
                out.record_stream(cout)
            routing.append((idx, gates, cnt))
        cur.wait_stream(cout)
        return routing

    # -- controller over the global batch (router.hpp:144-176, 158-169) --------
    def controller_step(self, idx: torch.Tensor, T: int, update: bool = True,
                        want_delta: bool = True):
        self.stream.wait_stream(torch.cuda.current_stream())
        delta = np.empty(self.shape.E, np.float64) if (update and want_delta) else None
        self.ctx._check(lib().scmoe_ep_controller_step(
            self.ep, self.router, idx.data_ptr(), T, int(update),
            None if delta is None else delta.ctypes.data_as(_P)))
        idx.record_stream(self.stream)
        return delta

    # -- state / stats -------------------------------------------------------------
    def bias(self) -> np.ndarray:
        b = np.empty(self.shape.E, np.float64)
        self.ctx._check(lib().scmoe_router_get_bias_host(self.ctx.handle, self.router,
                                                         b.ctypes.data_as(_P)))
        return b

    def count_matrix(self) -> np.ndarray:
        m = np.empty((self.world, self.world), np.int32)
        self.ctx._check(lib().scmoe_ep_count_matrix_host(self.ep, m.ctypes.data_as(_P)))
        return m

    def kernel_launches(self) -> int:
        """Kernels launched by the layer's contexts (the caller's + internal)."""
        return int(lib().scmoe_ep_kernel_launches(self.ep))

    def capacity_rows(self) -> int:
        return int(lib().scmoe_ep_capacity_rows(self.ep))

    def synchronize(self):
        self.ctx.synchronize()

    def close(self):
        L = lib()
        if self.ep:
            L.scmoe_ep_destroy(self.ep)
            self.ep = _P()
        if self.dense_bank:
            L.scmoe_bank_destroy(self.ctx.handle, self.dense_bank)
            self.dense_bank = None
        if self.bank:
            L.scmoe_bank_destroy(self.ctx.handle, self.bank)
            self.bank = _P()
        if self.router:
            L.scmoe_router_destroy(self.ctx.handle, self.router)
            self.router = _P()
