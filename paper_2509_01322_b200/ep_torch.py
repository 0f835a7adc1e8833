"""Expert-parallel ScMoE layer orchestrated in torch.distributed (reference
orchestration; the product path is the device-resident one in ep.py over the
C ABI, scmoe_ep_*).  Kept as the CPU-testable restatement of the dispatch plan
(tests/test_ep_gloo.py, gloo world 2) and as a NCCL-transport cross-check.

Partitioning: router + bias replicated on every rank, tokens sharded, FFN
experts block-partitioned (rank g owns [g*N/G, (g+1)*N/G)), zero experts
handled locally with no communication.  Per layer:

    1. route      rmsnorm + exact router + top-K on the local tokens
    2. plan       FFN slots grouped by owning rank, (token, slot) order
    3. counts     all-to-all of per-rank slot counts (G ints)
    4. dispatch   all-to-all of the slots' bf16 rows (+ their expert ids)
    5. experts    grouped GEMM1(+SiLU)/GEMM2 on the received rows (tcgen05)
    6. return     all-to-all of the expert output rows, in received order
    7. combine    rank-order combine + zero-expert identity + residual

With the dense shortcut branch enabled (GpuOps.enable_dense, SURVEY.md 8f1 /
config D) the layer also computes dd = a1 + ffn_block(rmsnorm(a1))
(model.hpp:390-391) on a second context and stream, concurrently with steps
1-6 -- the ScMoE overlap window: the dispatch and return all-to-alls hide
under the dense GEMMs -- and dd is the residual of step 7 (the second MLA,
model.hpp:392-393, is out of scope, so a3 = dd).  Its GEMMs are capped below
the SM count so the NCCL kernels always find free SMs.

Expert rows are returned per slot and combined at the source in the
reference's rank order (blocks.hpp:251-274), so the G-rank output is bitwise
equal to the single-GPU output.  The transport is torch.distributed's NCCL
all_to_all_single over NVLink/NVSwitch (plumbing); the numeric steps are the
C-ABI kernels, reached through a small ``ops`` object so that the
orchestration itself can be exercised on CPU with the gloo backend by the
tests (tests/test_ep_gloo.py) -- the product path always uses ``GpuOps``.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch
import torch.distributed as dist

from . import _P, Context, lib
from .layer import DenseFFN, LayerShape


class GpuOps:
    """The device kernels of one rank (C ABI), on torch CUDA tensors."""

    def __init__(self, ctx: Context, shape: LayerShape, rank: int, world: int, seed: int):
        self.ctx, self.shape, self.rank, self.world = ctx, shape, rank, world
        # kernels and NCCL collectives must be ordered on one stream: the layer
        # runs on this stream, made torch's current stream during forward()
        # (collectives synchronise with the current stream).  A real stream is
        # needed: handle 0 would select the context's private stream.
        self.stream = torch.cuda.Stream()
        ctx.set_stream(self.stream.cuda_stream)
        L = lib()
        s = shape
        if s.n_ffn % world:
            raise ValueError("world size must divide the FFN expert count")
        self.n_local = s.n_ffn // world
        self.first = rank * self.n_local
        self.router = _P()
        ctx._check(L.scmoe_router_create(ctx.handle, s.d, s.n_ffn, s.n_zero, s.top_k,
                                         s.k_expected, 0.0, 1.0, C.byref(self.router)))
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

    def _chk(self, rc):
        self.ctx._check(rc)

    def enable_dense(self, device: int, inter: int, seed: int, reserve_sms: int = 16):
        """Dense shortcut FFN on its own context + stream; its persistent GEMMs
        leave `reserve_sms` SMs to the communication kernels."""
        sms = torch.cuda.get_device_properties(device).multi_processor_count
        self.dense_ctx = Context(device)
        self.dense_stream = torch.cuda.Stream()
        self.dense_ctx.set_stream(self.dense_stream.cuda_stream)
        self.dense_ctx.set_sm_budget(0, max(1, sms - reserve_sms))
        self.dense = DenseFFN(self.dense_ctx, self.shape.d, inter, seed=seed)
        self.dense_ctx.synchronize()

    def dense_forward(self, a1: torch.Tensor, gain: Optional[torch.Tensor], T: int):
        """dd = a1 + ffn_block(rmsnorm(a1)) on the dense stream (not waited)."""
        self.dense_stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.dense_stream):
            dd = torch.empty(T, self.shape.d, dtype=torch.float32, device="cuda")
            self.dense.forward(a1.data_ptr(), None if gain is None else gain.data_ptr(), T,
                               dd.data_ptr())
        dd.record_stream(self.stream)  # consumed by the combine on the layer's stream
        return dd

    # -- peer-memory transport (NVLink; torch symmetric memory as the mapping) --
    def p2p_buffers(self, group, cap_recv: int, cap_send: int, nsets: int = 1):
        """(Re)allocates `nsets` sets of symmetric receive / receive-back buffers
        (collective: every rank calls it with the same capacities)."""
        import torch.distributed._symmetric_memory as symm_mem
        group = group if group is not None else dist.group.WORLD
        d = self.shape.d
        dev = lambda xs: torch.tensor(list(xs), dtype=torch.int64, device="cuda")  # noqa: E731
        self.p2p_cap = (cap_recv, cap_send)
        self.p2p_sets = []
        for _ in range(nsets):
            st = dict(recv=symm_mem.empty((cap_recv, d), dtype=torch.bfloat16, device="cuda"),
                      recv_exp=symm_mem.empty(cap_recv, dtype=torch.int32, device="cuda"),
                      back=symm_mem.empty((cap_send, d), dtype=torch.bfloat16, device="cuda"))
            st["h_recv"] = symm_mem.rendezvous(st["recv"], group)
            st["h_exp"] = symm_mem.rendezvous(st["recv_exp"], group)
            st["h_back"] = symm_mem.rendezvous(st["back"], group)
            st["peer_recv"] = dev(st["h_recv"].buffer_ptrs)
            st["peer_exp"] = dev(st["h_exp"].buffer_ptrs)
            st["peer_back"] = dev(st["h_back"].buffer_ptrs)
            self.p2p_sets.append(st)

    def put_rows(self, st, hb, send_token, send_expert, n_send, send_start, dst_offset):
        self._chk(lib().scmoe_ep_put_rows(self.ctx.handle, hb.data_ptr(), self.shape.d,
                                          send_token.data_ptr(), send_expert.data_ptr(), n_send,
                                          send_start.data_ptr(), dst_offset.data_ptr(),
                                          st["peer_recv"].data_ptr(), st["peer_exp"].data_ptr(),
                                          self.world))

    def experts_to(self, st, n_recv: int, row_dst: torch.Tensor, ctx: Optional[Context] = None):
        c = ctx or self.ctx
        c._check(lib().scmoe_moe_rows_to(c.handle, self.bank, st["recv"].data_ptr(),
                                         st["recv_exp"].data_ptr(), self.first, n_recv,
                                         row_dst.data_ptr()))

    def enable_back_context(self, device: int):
        """A second context + stream for the back half (expert GEMMs, combine) of
        the pipelined batch stream: its own workspace, so batch i's back half
        and batch i+1's front half never share scratch buffers."""
        if getattr(self, "ctx_b", None) is None:
            self.ctx_b = Context(device)
            self.stream_b = torch.cuda.Stream()
            self.ctx_b.set_stream(self.stream_b.cuda_stream)

    # -- load-balancing controller (router.hpp:144-176) over the global batch --
    def counters(self):
        import numpy as np
        E = self.shape.E
        r = np.empty(E, np.uint64)
        seen = C.c_uint64()
        self._chk(lib().scmoe_router_get_counters_host(self.ctx.handle, self.router,
                                                       r.ctypes.data_as(_P), C.byref(seen)))
        return r, int(seen.value)

    def set_counters(self, routed, seen: int):
        import numpy as np
        r = np.ascontiguousarray(routed, np.uint64)
        self._chk(lib().scmoe_router_set_counters_host(self.ctx.handle, self.router,
                                                       r.ctypes.data_as(_P), seen))

    def accumulate(self, idx: torch.Tensor, T: int):
        self._chk(lib().scmoe_accumulate_counters(self.ctx.handle, self.router, idx.data_ptr(), T))

    def bias_update(self):
        import numpy as np
        delta = np.empty(self.shape.E, np.float64)
        self._chk(lib().scmoe_bias_update(self.ctx.handle, self.router, delta.ctypes.data_as(_P)))
        return delta

    def bias(self):
        import numpy as np
        b = np.empty(self.shape.E, np.float64)
        self._chk(lib().scmoe_router_get_bias_host(self.ctx.handle, self.router,
                                                   b.ctypes.data_as(_P)))
        return b

    def route(self, a1: torch.Tensor, gain: Optional[torch.Tensor], T: int):
        s = self.shape
        hmoe = torch.empty(T, s.d, dtype=torch.float32, device="cuda")
        hb = torch.empty(T, s.d, dtype=torch.bfloat16, device="cuda")
        idx = torch.empty(T * s.top_k, dtype=torch.int32, device="cuda")
        gates = torch.empty(T * s.top_k, dtype=torch.float64, device="cuda")
        cnt = torch.empty(T, dtype=torch.int32, device="cuda")
        self._chk(lib().scmoe_rmsnorm_route(self.ctx.handle, self.router, a1.data_ptr(),
                                            None if gain is None else gain.data_ptr(), T,
                                            hmoe.data_ptr(), hb.data_ptr(), idx.data_ptr(),
                                            gates.data_ptr(), cnt.data_ptr()))
        return hmoe, hb, idx, gates, cnt

    def plan(self, idx: torch.Tensor, T: int):
        s = self.shape
        n = T * s.top_k
        counts = torch.empty(self.world, dtype=torch.int32, device="cuda")
        slot_pos = torch.empty(n, dtype=torch.int32, device="cuda")
        send_token = torch.empty(n, dtype=torch.int32, device="cuda")
        send_expert = torch.empty(n, dtype=torch.int32, device="cuda")
        self._chk(lib().scmoe_ep_plan(self.ctx.handle, idx.data_ptr(), T, s.top_k, s.n_ffn,
                                      s.n_zero, self.world, counts.data_ptr(), slot_pos.data_ptr(),
                                      send_token.data_ptr(), send_expert.data_ptr()))
        return counts, slot_pos, send_token, send_expert

    def gather(self, src: torch.Tensor, rows: torch.Tensor, n_rows: int):
        out = torch.empty(n_rows, self.shape.d, dtype=src.dtype, device="cuda")
        self._chk(lib().scmoe_gather_rows_bf16(self.ctx.handle, src.data_ptr(), self.shape.d,
                                               rows.data_ptr(), n_rows, out.data_ptr()))
        return out

    def experts(self, rows: torch.Tensor, row_expert: torch.Tensor):
        R = rows.shape[0]
        y = torch.empty_like(rows)
        self._chk(lib().scmoe_moe_rows(self.ctx.handle, self.bank, rows.data_ptr(),
                                       row_expert.data_ptr(), self.first, R, y.data_ptr()))
        return y

    def combine(self, hmoe, y_rows, slot_pos, idx, gates, T, a3, renormalize=False, ctx=None):
        s = self.shape
        c = ctx or self.ctx
        out = torch.empty(T, s.d, dtype=torch.float32, device="cuda")
        c._check(lib().scmoe_combine_rows(c.handle, self.bank, hmoe.data_ptr(),
                                           y_rows.data_ptr(), slot_pos.data_ptr(), idx.data_ptr(),
                                           gates.data_ptr(), T, s.top_k, s.n_ffn, int(renormalize),
                                           None if a3 is None else a3.data_ptr(), out.data_ptr()))
        return out

    def sync(self):
        torch.cuda.current_stream().synchronize()
        self.ctx.synchronize()

    def close(self):
        L = lib()
        if getattr(self, "dense", None) is not None:
            self.dense.close()
            self.dense = None
        L.scmoe_bank_destroy(self.ctx.handle, self.bank)
        L.scmoe_router_destroy(self.ctx.handle, self.router)


class EPLayer:
    """One ScMoE MoE branch sharded over the ranks of ``group``."""

    def __init__(self, ops, group=None, async_comm: bool = True, transport: str = "nccl"):
        """transport "nccl": all_to_all_single for the rows; "p2p": the rows are
        stored straight into the peers' symmetric buffers over NVLink by the
        dispatch kernel and by GEMM2's epilogue (return fused into the GEMM)."""
        self.ops, self.group = ops, group
        self.async_comm = async_comm
        if transport not in ("nccl", "p2p"):
            raise ValueError("transport must be 'nccl' or 'p2p'")
        self.transport = transport
        # comm=False replaces the row all-to-alls by no-ops (receive buffers left
        # uninitialised): the timing reference for the exposed-communication share
        self.comm = True
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.last_stats = {}

    def forward(self, a1: torch.Tensor, a3: Optional[torch.Tensor], gain, T: int,
                renormalize: bool = False, chunks: int = 1, dense: bool = False):
        """chunks > 1 splits the tokens into micro-chunks processed as a
        software pipeline: chunk c+1's routing runs while chunk
        c's rows are in flight, chunk c's expert GEMMs while chunk c+1's rows
        are in flight, and so on.  Results are bitwise identical to chunks=1
        (every step is per-token independent).  dense=True runs the dense
        shortcut branch concurrently and uses dd as the residual (a3 ignored)."""
        stream = getattr(self.ops, "stream", None)
        if stream is None:
            return self._forward(a1, a3, gain, T, renormalize, chunks)
        # inputs produced on the caller's stream must be complete first
        stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(stream):
            dd = self.ops.dense_forward(a1, gain, T) if dense else None
            res = self._forward(a1, dd if dense else a3, gain, T, renormalize, chunks,
                                wait_residual=self.ops.dense_stream if dense else None)
        torch.cuda.current_stream().wait_stream(stream)
        for t in res:
            t.record_stream(torch.cuda.current_stream())
        return res

    # -- pipeline stages (all on the current stream; collectives async) -------
    def _dispatch(self, a1, gain, t0, t1):
        ops, G = self.ops, self.world
        T = t1 - t0
        a1c = a1.reshape(-1)[t0 * self.d:t1 * self.d]
        hmoe, hb, idx, gates, cnt = ops.route(a1c, gain, T)
        counts, slot_pos, send_token, send_expert = ops.plan(idx, T)
        # count exchange (G ints); split sizes are needed on the host
        recv_counts = torch.empty_like(counts)
        dist.all_to_all_single(recv_counts, counts, group=self.group)
        both = torch.cat([counts, recv_counts]).cpu().tolist()
        send_split, recv_split = both[:G], both[G:]
        n_send, n_recv = sum(send_split), sum(recv_split)
        send_rows = ops.gather(hb, send_token, n_send)
        recv_rows = torch.empty(n_recv, hb.shape[1], dtype=hb.dtype, device=hb.device)
        recv_expert = torch.empty(n_recv, dtype=send_expert.dtype, device=send_expert.device)
        if self.comm:
            w_rows = dist.all_to_all_single(recv_rows, send_rows, recv_split, send_split,
                                            group=self.group, async_op=self.async_comm)
            w_exp = dist.all_to_all_single(recv_expert, send_expert[:n_send].contiguous(),
                                           recv_split, send_split, group=self.group,
                                           async_op=self.async_comm)
        else:  # timing reference: received rows are garbage, expert ids valid
            recv_expert.fill_(ops.first if hasattr(ops, "first") else 0)
            w_rows = w_exp = None
        return dict(t0=t0, T=T, hmoe=hmoe, idx=idx, gates=gates, cnt=cnt, slot_pos=slot_pos,
                    send_split=send_split, recv_split=recv_split, n_send=n_send, n_recv=n_recv,
                    recv_rows=recv_rows, recv_expert=recv_expert, waits=[w_rows, w_exp],
                    keep=[send_rows], width=hb.shape[1], dtype=hb.dtype)

    def _experts(self, st):
        for w in st.pop("waits"):
            if w is not None:
                w.wait()
        y_rows = self.ops.experts(st["recv_rows"], st["recv_expert"])
        back = torch.empty(st["n_send"], st["width"], dtype=st["dtype"], device=y_rows.device)
        st["w_back"] = (dist.all_to_all_single(back, y_rows, st["send_split"], st["recv_split"],
                                               group=self.group, async_op=self.async_comm)
                        if self.comm else None)
        st["back"] = back
        st["keep"].append(y_rows)

    def _combine(self, st, a3, renormalize, wait_residual=None):
        w = st.pop("w_back")
        if w is not None:
            w.wait()
        if wait_residual is not None:  # dd from the dense stream
            torch.cuda.current_stream().wait_stream(wait_residual)
        a3c = None if a3 is None else a3.view(-1)[st["t0"] * self.d:(st["t0"] + st["T"]) * self.d]
        return self.ops.combine(st["hmoe"], st["back"], st["slot_pos"], st["idx"], st["gates"],
                                st["T"], a3c, renormalize)

    def _front_p2p(self, a1, gain, T, nsets=1, k=0):
        """Route, plan, counts all-gather (host sync) and the dispatch into the
        owners' receive buffers of set k, then a cross-rank barrier."""
        ops, G, me = self.ops, self.world, self.rank
        hmoe, hb, idx, gates, cnt = ops.route(a1, gain, T)
        counts, slot_pos, send_token, send_expert = ops.plan(idx, T)
        # full [src][dst] slot-count matrix on every rank: offsets + capacities
        allc = torch.empty(G * G, dtype=counts.dtype, device=counts.device)
        dist.all_gather_into_tensor(allc, counts, group=self.group)
        Mh = allc.view(G, G).cpu().tolist()
        n_send = sum(Mh[me])
        n_recv = sum(Mh[s][me] for s in range(G))
        need_r = max(sum(Mh[s][d] for s in range(G)) for d in range(G))
        need_s = max(sum(r) for r in Mh)
        cap = getattr(ops, "p2p_cap", (0, 0))
        if (need_r > cap[0] or need_s > cap[1]
                or len(getattr(ops, "p2p_sets", [])) < nsets):  # same decision on every rank
            torch.cuda.synchronize()  # no set may be in use while it is replaced
            ops.p2p_buffers(self.group, max(1, int(max(need_r, cap[0]) * 1.25)),
                            max(1, int(max(need_s, cap[1]) * 1.25)), nsets=max(nsets, 1))
        st = ops.p2p_sets[k]
        # offsets from the count matrix, on the device (no per-step host copies)
        Md = allc.view(G, G).to(torch.int64)
        col_excl = torch.cumsum(Md, 0) - Md            # [s][d] = sum_{s'<s} M[s'][d]
        row_excl = torch.cumsum(Md, 1) - Md            # [s][d] = sum_{d'<d} M[s][d']
        send_start = torch.zeros(G + 1, dtype=torch.int32, device=Md.device)
        send_start[1:] = torch.cumsum(Md[me], 0).to(torch.int32)
        dst_offset = col_excl[me].contiguous()         # where my rows start in rank d's buffer
        recv_offset = col_excl[:, me]                  # where source s's rows start in mine
        back_start = row_excl[:, me]                   # source s's send index of its rows for me
        dev = counts.device
        src = torch.repeat_interleave(torch.arange(G, device=dev), Md[:, me], output_size=n_recv)
        j = torch.arange(n_recv, dtype=torch.int64, device=dev) - recv_offset[src]
        # received row r (source s's j-th row for me) returns to source s's back
        # buffer at row back_start[s] + j; comm=False (timing reference): no
        # dispatch, GEMM2 rows stay local
        back_ptr = st["peer_back"] if self.comm else \
            torch.full_like(st["peer_back"], st["back"].data_ptr())
        row_dst = back_ptr[src] + (back_start[src] + j) * (ops.shape.d * 2)
        if self.comm:
            ops.put_rows(st, hb, send_token, send_expert, n_send, send_start, dst_offset)
        else:
            st["recv_exp"][:n_recv].fill_(ops.first)
        st["h_recv"].barrier(channel=0)
        return dict(k=k, T=T, hmoe=hmoe, idx=idx, gates=gates, cnt=cnt, slot_pos=slot_pos,
                    n_send=n_send, n_recv=n_recv, self_rows=Mh[me][me], row_dst=row_dst,
                    keep=[hb, send_token,
                                                                        send_expert])

    def _back_p2p(self, f, a3, renormalize, wait_residual=None, ctx=None):
        """Expert GEMMs on the received rows (GEMM2 rows land in the sources'
        back buffers), barrier, rank-order combine."""
        ops = self.ops
        st = ops.p2p_sets[f["k"]]
        ops.experts_to(st, f["n_recv"], f["row_dst"], ctx=ctx)
        st["h_back"].barrier(channel=1)
        if wait_residual is not None:
            torch.cuda.current_stream().wait_stream(wait_residual)
        return ops.combine(f["hmoe"], st["back"], f["slot_pos"], f["idx"], f["gates"], f["T"], a3,
                           renormalize, ctx=ctx)

    def _forward_p2p(self, a1, a3, gain, T, renormalize, wait_residual=None):
        """One chunk, peer-memory transport (see __init__)."""
        f = self._front_p2p(a1, gain, T)
        out = self._back_p2p(f, a3, renormalize, wait_residual)
        self.last_stats = {"send_rows": f["n_send"], "recv_rows": f["n_recv"], "chunks": 1,
                           "transport": "p2p", "self_rows": f["self_rows"],
                           "a2a_bytes_each_way": f["n_send"] * self.ops.shape.d * 2}
        return out, f["idx"], f["gates"], f["cnt"]

    def controller_step(self, idx: torch.Tensor, T: int, update: bool = True):
        """accumulate_counters for this rank's routing, then (update=True) the
        PID bias update over the GLOBAL batch: the per-expert
        slot counters and tokens_seen are summed over the ranks (exact
        integers), so every rank applies the same bias_update -- identical to a
        single router that routed all ranks' tokens.  Returns the deltas."""
        ops = self.ops
        stream = getattr(ops, "stream", None)
        if stream is not None:
            stream.wait_stream(torch.cuda.current_stream())
        ops.accumulate(idx, T)
        if not update:
            return None
        routed, seen = ops.counters()  # synchronises the context's stream
        t = torch.tensor(list(routed.astype("int64")) + [seen], dtype=torch.int64, device="cuda")
        dist.all_reduce(t, group=self.group)
        tot = t.cpu().tolist()
        ops.set_counters(tot[:-1], tot[-1])
        return ops.bias_update()

    def forward_host_batches(self, a1s, a3s, outs, gain, T: int, renormalize: bool = False):
        """Host tier for a stream of batches (pinned host tensors a1s / a3s in,
        outs filled): the copy-in of batch i+1 and the copy-out of batch i-1
        run on copy streams while batch i computes (device inputs double
        buffered).  Returns the routing of every batch (device tensors)."""
        stream = getattr(self.ops, "stream", torch.cuda.current_stream())
        cin, cout = torch.cuda.Stream(), torch.cuda.Stream()
        n = len(a1s)
        dev = [dict(a1=torch.empty(a1s[0].shape, dtype=a1s[0].dtype, device="cuda"),
                    a3=None if a3s is None else torch.empty(a3s[0].shape, dtype=a3s[0].dtype,
                                                           device="cuda")) for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(n)]
        ev_used = [torch.cuda.Event() for _ in range(n)]
        caller = torch.cuda.current_stream()
        cin.wait_stream(caller)
        cout.wait_stream(caller)

        def copy_in(i):
            with torch.cuda.stream(cin):
                if i >= 2:
                    cin.wait_event(ev_used[i - 2])  # the slot's inputs were read by batch i-2
                b = dev[i % 2]
                b["a1"].copy_(a1s[i], non_blocking=True)
                if a3s is not None:
                    b["a3"].copy_(a3s[i], non_blocking=True)
                ev_in[i].record(cin)

        routing = []
        copy_in(0)
        for i in range(n):
            if i + 1 < n:
                copy_in(i + 1)  # issued before forward(i), whose host sync would delay it
            caller.wait_event(ev_in[i])
            b = dev[i % 2]
            out, idx, gates, cnt = self.forward(b["a1"], b["a3"], gain, T, renormalize)
            ev_used[i].record(caller)
            with torch.cuda.stream(cout):
                cout.wait_event(ev_used[i])
                outs[i].copy_(out.view(outs[i].shape), non_blocking=True)
                out.record_stream(cout)
            routing.append((idx, gates, cnt))
        caller.wait_stream(cout)
        return routing

    def forward_batches(self, a1s, a3s, gain, T: int, renormalize: bool = False,
                        corun_router: bool = False):
        """A stream of batches, pipelined (p2p transport): batch i+1's front half
        (routing, planning, dispatch over NVLink) runs on the front stream while batch i's
        expert GEMMs + return + combine run on the back stream / context.  Two
        sets of symmetric buffers alternate.  Results equal len(a1s) forward()
        calls bit for bit.  corun_router selects the small router kernel that
        co-resides with the GEMM (faster at N=1's HBM-bound GEMMs; at EP shapes
        the GEMMs lean on the tensor pipe and the full-size router, which
        time-shares the SMs instead, measured faster)."""
        if self.transport != "p2p":
            raise ValueError("forward_batches needs the p2p transport")
        ops = self.ops
        dev = torch.cuda.current_device()
        ops.enable_back_context(dev)
        F, B = ops.stream, ops.stream_b
        caller = torch.cuda.current_stream()
        F.wait_stream(caller)
        B.wait_stream(caller)
        ops.ctx.set_overlapped(corun_router)
        n = len(a1s)
        fronts, outs = [None] * n, [None] * n
        ev_front = [torch.cuda.Event() for _ in range(n)]
        ev_back = [torch.cuda.Event() for _ in range(n)]
        try:
            for i in range(n + 1):
                if i >= 1:  # back(i-1) first, so the GPU has it before the host blocks
                    with torch.cuda.stream(B):
                        B.wait_event(ev_front[i - 1])
                        outs[i - 1] = self._back_p2p(fronts[i - 1],
                                                     None if a3s is None else a3s[i - 1],
                                                     renormalize, ctx=ops.ctx_b)
                        ev_back[i - 1].record(B)
                if i < n:
                    with torch.cuda.stream(F):
                        if i >= 2:  # set i % 2 was last used by batch i-2
                            F.wait_event(ev_back[i - 2])
                        fronts[i] = self._front_p2p(a1s[i], gain, T, nsets=2, k=i % 2)
                        ev_front[i].record(F)
        finally:
            ops.ctx.set_overlapped(False)
        caller.wait_stream(B)
        caller.wait_stream(F)
        res = []
        for i in range(n):
            for t in (outs[i], fronts[i]["idx"], fronts[i]["gates"], fronts[i]["cnt"]):
                t.record_stream(caller)
            res.append((outs[i], fronts[i]["idx"], fronts[i]["gates"], fronts[i]["cnt"]))
        f = fronts[-1]
        self.last_stats = {"send_rows": f["n_send"], "recv_rows": f["n_recv"], "chunks": 1,
                           "transport": "p2p", "pipelined": True, "self_rows": f["self_rows"],
                           "a2a_bytes_each_way": f["n_send"] * ops.shape.d * 2}
        return res

    def _forward(self, a1, a3, gain, T, renormalize, chunks, wait_residual=None):
        self.d = self.ops.shape.d if hasattr(self.ops, "shape") else a1.numel() // T
        if self.transport == "p2p":
            return self._forward_p2p(a1, a3, gain, T, renormalize, wait_residual)
        chunks = max(1, min(chunks, T))
        bounds = [T * c // chunks for c in range(chunks + 1)]
        # issue order: D0 D1 E0 D2 E1 C0 ... so each collective has independent
        # compute queued behind it on the GPU
        states = []
        outs = []
        for c in range(chunks + 2):
            if c < chunks:
                states.append(self._dispatch(a1, gain, bounds[c], bounds[c + 1]))
            if 0 <= c - 1 < chunks:
                self._experts(states[c - 1])
            if 0 <= c - 2 < chunks:
                outs.append(self._combine(states[c - 2], a3, renormalize, wait_residual))
        n_send = sum(s["n_send"] for s in states)
        n_recv = sum(s["n_recv"] for s in states)
        self.last_stats = {"send_rows": n_send, "recv_rows": n_recv, "chunks": chunks,
                           "a2a_bytes_each_way": n_send * states[0]["width"] * 2}
        cat = lambda key: torch.cat([s[key] for s in states]) if chunks > 1 else states[0][key]  # noqa: E731
        out = torch.cat([o.view(-1) for o in outs]).view(T, -1) if chunks > 1 else outs[0]
        return out, cat("idx"), cat("gates"), cat("cnt")
