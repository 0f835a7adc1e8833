"""Expert parallelism on real GPUs (NCCL over NVLink): the G-rank EP layer's
routing and output are bitwise equal to the single-GPU layer on the same
tokens (per-slot expert rows, rank-order combine at the source)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q, chunks=1, dense=False, transport="nccl", renorm=False):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        import paper_2509_01322_b200 as P
        from paper_2509_01322_b200.ep import EPLayer, GpuOps
        from paper_2509_01322_b200.layer import DeviceLayer, LayerShape
        shape = LayerShape(d=1024, n_ffn=64, n_zero=32, top_k=6, k_expected=4, inter=512,
                           precision=P.PREC_BF16)
        T = 640 + 64 * rank  # ragged shards
        a1 = torch.from_numpy(P.fill_normal(P.stream_seed(9, rank), T * shape.d)).cuda()
        a3 = torch.from_numpy(P.fill_normal(P.stream_seed(10, rank), T * shape.d)).cuda()
        ctx = P.Context(rank)
        ops = GpuOps(ctx, shape, rank, world, seed=3)
        if dense:
            ops.enable_dense(rank, inter=1024, seed=7)
        ep = EPLayer(ops, transport=transport)
        out, idx, gates, cnt = ep.forward(a1, a3, None, T, chunks=chunks, dense=dense,
                                          renormalize=renorm)
        torch.cuda.synchronize()
        # single-GPU reference: same seed => same router and the full expert set
        ctx1 = P.Context(rank)
        s1 = torch.cuda.Stream()
        ctx1.set_stream(s1.cuda_stream)
        full = DeviceLayer(ctx1, shape, seed=3)
        if dense:  # the dense branch's dd is the MoE residual (a3 = dd)
            from paper_2509_01322_b200.layer import DenseFFN
            dn = DenseFFN(ctx1, shape.d, 1024, seed=7)
            a3 = torch.empty_like(a1)
            dn.forward(a1.data_ptr(), None, T, a3.data_ptr())
        idx1 = torch.empty_like(idx)
        gates1 = torch.empty_like(gates)
        cnt1 = torch.empty_like(cnt)
        out1 = torch.empty_like(out)
        full.forward(a1.data_ptr(), a3.data_ptr(), None, T, idx1.data_ptr(), gates1.data_ptr(),
                     cnt1.data_ptr(), out1.data_ptr(), renormalize=renorm)
        torch.cuda.synchronize()
        ok = (torch.equal(idx, idx1) and torch.equal(gates, gates1) and torch.equal(out, out1))
        info = dict(ep.last_stats, idx_diff=int((idx != idx1).sum()),
                    out_diff=int((out != out1).sum()),
                    rel=float((out - out1).norm() / out1.norm()))
        q.put((rank, bool(ok), info))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,chunks,dense,transport", [
    (1, 1, False, "nccl"), (2, 1, False, "nccl"), (2, 2, False, "nccl"), (4, 3, False, "nccl"),
    (1, 1, True, "nccl"), (2, 1, True, "nccl"), (4, 2, True, "nccl"),
    (1, 1, False, "p2p"), (2, 1, False, "p2p"), (4, 1, False, "p2p"), (2, 1, True, "p2p"),
    (4, 1, True, "p2p")])
def test_ep_equals_single_gpu_bitwise(world, chunks, dense, transport):
    import torch
    import torch.multiprocessing as mp
    n = torch.cuda.device_count()
    if n < world:
        pytest.skip(f"needs >= {world} GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 200
    port += chunks + 7 * dense + 17 * (transport == "p2p")
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, chunks, dense, transport))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, info in sorted(res):
        assert ok, f"rank {rank}: {info}"


def _batches_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        import paper_2509_01322_b200 as P
        from paper_2509_01322_b200.ep import EPLayer, GpuOps
        from paper_2509_01322_b200.layer import LayerShape
        shape = LayerShape(d=1024, n_ffn=64, n_zero=32, top_k=6, k_expected=4, inter=512,
                           precision=P.PREC_BF16)
        T, nb = 704 + 32 * rank, 4
        a1 = [torch.from_numpy(P.fill_normal(P.stream_seed(40 + i, rank), T * shape.d)).cuda()
              for i in range(nb)]
        a3 = [torch.from_numpy(P.fill_normal(P.stream_seed(50 + i, rank), T * shape.d)).cuda()
              for i in range(nb)]
        ep = EPLayer(GpuOps(P.Context(rank), shape, rank, world, seed=3), transport="p2p")
        ser = [ep.forward(a1[i], a3[i], None, T) for i in range(nb)]
        torch.cuda.synchronize()
        pip = ep.forward_batches(a1, a3, None, T)
        pip2 = ep.forward_batches(a1[:2], None, None, T)  # again, and without residual
        torch.cuda.synchronize()
        ok = all(torch.equal(u, v) for s, p in zip(ser, pip) for u, v in zip(s, p))
        ref2 = [ep.forward(a1[i], None, None, T)[0] for i in range(2)]
        torch.cuda.synchronize()
        ok = ok and all(torch.equal(r, p[0]) for r, p in zip(ref2, pip2))
        q.put((rank, bool(ok), ep.last_stats))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 4])
def test_ep_pipelined_batches_equal_serial(world):
    """EPLayer.forward_batches (front of batch i+1 beside the back of batch i,
    co-resident router, two symmetric buffer sets) == serial forward() calls."""
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs >= {world} GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29950 + world + os.getpid() % 40
    procs = [ctx.Process(target=_batches_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, info in sorted(res):
        assert ok, f"rank {rank}: {info}"


def _host_batches_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        import paper_2509_01322_b200 as P
        from paper_2509_01322_b200.ep import EPLayer, GpuOps
        from paper_2509_01322_b200.layer import LayerShape
        shape = LayerShape(d=1024, n_ffn=64, n_zero=32, top_k=6, k_expected=4, inter=512,
                           precision=P.PREC_BF16)
        T, nb = 512 + 64 * rank, 3
        a1 = [torch.from_numpy(P.fill_normal(P.stream_seed(70 + i, rank), T * shape.d)
                               .reshape(T, shape.d)).pin_memory() for i in range(nb)]
        a3 = [torch.from_numpy(P.fill_normal(P.stream_seed(80 + i, rank), T * shape.d)
                               .reshape(T, shape.d)).pin_memory() for i in range(nb)]
        ep = EPLayer(GpuOps(P.Context(rank), shape, rank, world, seed=3), transport="p2p")
        outs = [torch.empty(T, shape.d).pin_memory() for _ in range(nb)]
        ep.forward_host_batches(a1, a3, outs, None, T)
        torch.cuda.synchronize()
        ok = True
        for i in range(nb):
            ref = ep.forward(a1[i].cuda(), a3[i].cuda(), None, T)[0]
            torch.cuda.synchronize()
            ok = ok and torch.equal(ref.cpu(), outs[i])
        q.put((rank, bool(ok), ""))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_ep_host_batches_equal_device_calls():
    """EPLayer.forward_host_batches (copy streams, double-buffered inputs) returns
    exactly what per-batch device calls return."""
    import torch
    import torch.multiprocessing as mp
    world = min(2, torch.cuda.device_count())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29890 + os.getpid() % 40
    procs = [ctx.Process(target=_host_batches_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, info in sorted(res):
        assert ok, f"rank {rank}: {info}"


@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_ep_renormalised_gates_bitwise(transport):
    """Gate renormalisation (blocks.hpp:240-247) through the EP combine."""
    import torch
    import torch.multiprocessing as mp
    world = min(2, torch.cuda.device_count())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29810 + os.getpid() % 40 + (transport == "p2p")
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, 1, False, transport, True))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, info in sorted(res):
        assert ok, f"rank {rank}: {info}"


def _controller_worker(rank, world, port, q):
    import numpy as np
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        import paper_2509_01322_b200 as P
        from paper_2509_01322_b200.ep import EPLayer, GpuOps
        from paper_2509_01322_b200.layer import DeviceLayer, LayerShape
        shape = LayerShape(d=1024, n_ffn=64, n_zero=32, top_k=6, k_expected=3, inter=512,
                           precision=P.PREC_BF16)
        T = 512 + 128 * rank
        ops = GpuOps(P.Context(rank), shape, rank, world, seed=3)
        ep = EPLayer(ops, transport="p2p")
        # a controller that moves: mu > 0 on every rank's replica of the router
        lib = P.lib()
        ops.ctx._check(lib.scmoe_router_set_mu(ops.ctx.handle, ops.router, 0.2, 0.999))
        deltas, idxs = [], []
        for step in range(3):
            a1 = torch.from_numpy(P.fill_normal(P.stream_seed(90 + step, rank), T * shape.d)).cuda()
            out, idx, gates, cnt = ep.forward(a1, None, None, T)
            deltas.append(ep.controller_step(idx, T))
            # every rank's routing of this step, for the single-router reference
            sizes = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(world)]
            dist.all_gather(sizes, torch.tensor([idx.numel()], device="cuda"))
            parts = [torch.empty(int(s.item()), dtype=idx.dtype, device="cuda") for s in sizes]
            dist.all_gather(parts, idx)
            idxs.append([p_.cpu() for p_ in parts])
        torch.cuda.synchronize()
        # same bias on every rank
        b = torch.from_numpy(ops.bias()).cuda()
        b0 = b.clone()
        dist.broadcast(b0, 0)
        ok = torch.equal(b, b0)
        # single router fed every rank's slots in rank order: identical deltas
        ctx1 = P.Context(rank)
        ref = DeviceLayer(ctx1, shape, seed=3, mu=0.2, mu_decay=0.999)
        for step in range(3):
            for part in idxs[step]:
                ref.accumulate(part.cuda().data_ptr(), part.numel() // shape.top_k)
            d_ref = ref.bias_update()
            ok = ok and d_ref.tobytes() == deltas[step].tobytes()
        ok = ok and ref.bias().tobytes() == ops.bias().tobytes()
        q.put((rank, bool(ok), ""))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_ep_controller_global_batch_bitwise():
    """the bias controller under EP sums the per-expert counters
    and tokens over the ranks; every rank's bias_update equals one router's
    update over all ranks' slots, bit for bit."""
    import torch
    import torch.multiprocessing as mp
    world = min(2, torch.cuda.device_count())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29850 + os.getpid() % 40
    procs = [ctx.Process(target=_controller_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, info in sorted(res):
        assert ok, f"rank {rank}: {info}"
