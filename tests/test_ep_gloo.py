"""CPU test of the expert-parallel orchestration (paper_2509_01322_b200/ep_torch.py)
with world_size 2 over gloo.

The numeric steps are provided by an oracle-backed ``ops`` object (test
infrastructure, fp32), so the test checks exactly what ep_torch.py owns: the dispatch
plan order, count exchange, split sizes, expert-id localisation, the return
order of the expert rows and the source-side combine mapping.  The EP result
on each rank's token shard must equal the single-process oracle layer on the
same tokens bit for bit."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

D, N, Z, K, KE, I = 64, 8, 4, 3, 2, 32
T_LOCAL = 48
SEED_W, SEED_X = 5, 99


def _weights():
    import _oracle as O
    w_r = O.uniform_f32(O.stream_seed(SEED_W, 0), D * (N + Z), 1.0 / D).reshape(D, N + Z)
    w_in = [O.uniform_f32(O.stream_seed(SEED_W, 100 + 2 * e), D * I, 1.0 / D).reshape(D, I)
            for e in range(N)]
    w_out = [O.uniform_f32(O.stream_seed(SEED_W, 101 + 2 * e), I * D, 1.0 / D).reshape(I, D)
             for e in range(N)]
    return w_r, w_in, w_out


class OracleOps:
    """Oracle-backed stand-ins for GpuOps (fp32, exact reference arithmetic)."""

    def __init__(self, rank, world):
        import _oracle as O
        self.O = O
        self.rank, self.world = rank, world
        self.w_r, self.w_in, self.w_out = _weights()
        self.per = N // world
        self.first = rank * self.per

    def route(self, a1, gain, T):
        import torch
        O = self.O
        x = a1.numpy().reshape(T, D)
        g = np.ones(D, np.float32)
        h = np.empty_like(x)
        O.orc().orc_rmsnorm_f32(O.ptr(x), O.ptr(g), T, D, np.float32(1e-6), O.ptr(h))
        rc, idx, gates, cnt, _ = O.orc_route_topk(h, self.w_r, N, Z, K, KE)
        assert rc == 0
        ht = torch.from_numpy(h)
        return ht, ht, torch.from_numpy(idx.astype(np.int32)), torch.from_numpy(gates), \
            torch.from_numpy(cnt.astype(np.int32))

    def plan(self, idx, T):
        import torch
        idx = idx.numpy()
        dest_lists = [[] for _ in range(self.world)]
        for i, e in enumerate(idx):
            if e < N:
                dest_lists[e // self.per].append(i)
        slot_pos = np.full(T * K, -1, np.int32)
        send_token = np.zeros(T * K, np.int32)
        send_expert = np.zeros(T * K, np.int32)
        p = 0
        for lst in dest_lists:
            for i in lst:
                slot_pos[i] = p
                send_token[p] = i // K
                send_expert[p] = idx[i]
                p += 1
        counts = np.array([len(lst) for lst in dest_lists], np.int32)
        return (torch.from_numpy(counts), torch.from_numpy(slot_pos), torch.from_numpy(send_token),
                torch.from_numpy(send_expert))

    def gather(self, src, rows, n):
        return src[rows[:n].long()].contiguous()

    def experts(self, rows, row_expert):
        import torch
        O = self.O
        r = rows.numpy()
        y = np.empty_like(r)
        h = np.empty(I, np.float32)
        for j in range(r.shape[0]):
            e = int(row_expert[j])
            assert self.first <= e < self.first + self.per, "row sent to the wrong rank"
            O.orc().orc_expert_row_f32(O.ptr(r[j]), D, O.ptr(self.w_in[e]), O.ptr(self.w_out[e]), I,
                                       O.ptr(h), O.ptr(y[j]))
        return torch.from_numpy(y)

    def combine(self, hmoe, y_rows, slot_pos, idx, gates, T, a3, renormalize=False):
        import torch
        x = hmoe.numpy()
        y = y_rows.numpy()
        idx = idx.numpy()
        gates = gates.numpy()
        sp = slot_pos.numpy()
        out = np.zeros((T, D), np.float32)
        one = np.float32(1.0)
        for t in range(T):
            zero_w = np.float32(0.0)
            for s in range(K):
                e = idx[t * K + s]
                w = np.float32(gates[t * K + s]) / one
                if e < N:
                    out[t] = out[t] + (one * w) * y[sp[t * K + s]]
                else:
                    zero_w = np.float32(zero_w + w)
            if zero_w != 0:
                out[t] = out[t] + (one * zero_w) * x[t]
        if a3 is not None:
            out = a3.numpy().reshape(T, D) + out
        return torch.from_numpy(out.astype(np.float32))


def _worker(rank, world, port, q, chunks=1):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import _oracle as O
        from paper_2509_01322_b200.ep_torch import EPLayer
        a1 = torch.from_numpy(O.normal_f32(O.stream_seed(SEED_X, rank), T_LOCAL * D))
        a3 = torch.from_numpy(O.normal_f32(O.stream_seed(SEED_X + 1, rank), T_LOCAL * D))
        layer = EPLayer(OracleOps(rank, world))
        out, idx, gates, cnt = layer.forward(a1, a3, None, T_LOCAL, chunks=chunks)
        # single-process oracle on this rank's tokens
        w_r, w_in, w_out = _weights()
        want = np.empty((T_LOCAL, D), np.float32)
        wi = np.empty(T_LOCAL * K, np.uint32)
        wg = np.empty(T_LOCAL * K)
        wc = np.empty(T_LOCAL, np.uint32)
        rc = O.orc().orc_scmoe_layer_f32(O.ptr(a1.numpy()), O.ptr(a3.numpy()),
                                         O.ptr(np.ones(D, np.float32)), T_LOCAL, D, O.ptr(w_r), N,
                                         Z, K, KE, 0.0, O.ptr(np.zeros(N + Z)), O.ptr_array(w_in),
                                         O.ptr_array(w_out), I, 1.0, 1.0, 0, O.ptr(wi), O.ptr(wg),
                                         O.ptr(wc), O.ptr(want))
        ok = (rc == 0 and (idx.numpy().astype(np.uint32) == wi).all() and
              (out.numpy().view(np.uint32) == want.view(np.uint32)).all())
        q.put((rank, bool(ok), layer.last_stats))
    except Exception as e:  # pragma: no cover - surfaced through the queue
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,chunks", [(2, 1), (2, 3)])
def test_ep_orchestration_gloo(world, chunks):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 200
    procs = [ctx.Process(target=_worker, args=(r, world, port + chunks, q, chunks))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, info in sorted(res):
        assert ok, f"rank {rank}: {info}"
    sent = sum(info["send_rows"] for _, _, info in res)
    recv = sum(info["recv_rows"] for _, _, info in res)
    assert sent == recv > 0
