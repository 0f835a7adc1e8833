"""Expert parallelism on real GPUs: the device-resident C-ABI orchestration
(scmoe_ep_*, csrc/ep.cu; Python caller paper_2509_01322_b200/ep.py).

The G-rank layer's routing and output are bitwise equal to the single-GPU
layer on the same tokens (per-slot expert rows, rank-order combine at the
source), for ragged per-rank token counts, with and without the dense
shortcut branch and gate renormalisation, serial and pipelined; the
controller's bias update over the global batch equals one router fed every
rank's slots.  World sizes above the box's GPU count are skipped.  One case
cross-checks the torch.distributed reference orchestration (ep_torch.py)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


def _spawn(target, world, port, *args):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs >= {world} GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=900) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, ok, info in sorted(res, key=lambda r: r[0]):
        assert ok, f"rank {rank}: {info}"
    return res


def _init(rank, world, port):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)  # id hand-off only


def _shape(P, ke=4):
    from paper_2509_01322_b200.layer import LayerShape
    return LayerShape(d=1024, n_ffn=64, n_zero=32, top_k=6, k_expected=ke, inter=512,
                      precision=P.PREC_BF16)


def _single_gpu(P, rank, shape, a1, a3, T, renorm=False, dense_inter=0):
    """The single-GPU layer (full expert set, same seeds) on the same tokens."""
    import torch
    from paper_2509_01322_b200.layer import DenseFFN, DeviceLayer
    ctx1 = P.Context(rank)
    s1 = torch.cuda.Stream()
    ctx1.set_stream(s1.cuda_stream)
    full = DeviceLayer(ctx1, shape, seed=3)
    if dense_inter:  # dd is the MoE residual (a3 = dd)
        dn = DenseFFN(ctx1, shape.d, dense_inter, seed=7)
        a3 = torch.empty_like(a1)
        dn.forward(a1.data_ptr(), None, T, a3.data_ptr())
    out = torch.empty(T, shape.d, device="cuda")
    idx = torch.empty(T * shape.top_k, dtype=torch.int32, device="cuda")
    gates = torch.empty(T * shape.top_k, dtype=torch.float64, device="cuda")
    cnt = torch.empty(T, dtype=torch.int32, device="cuda")
    full.forward(a1.data_ptr(), None if a3 is None else a3.data_ptr(), None, T, idx.data_ptr(),
                 gates.data_ptr(), cnt.data_ptr(), out.data_ptr(), renormalize=renorm)
    ctx1.synchronize()
    return out, idx, gates, cnt


def _equal_worker(rank, world, port, q, dense, renorm):
    import torch
    import torch.distributed as dist
    _init(rank, world, port)
    try:
        import paper_2509_01322_b200 as P
        from paper_2509_01322_b200.ep import ExpertParallelLayer, broadcast_unique_id
        shape = _shape(P)
        T = 640 + 64 * rank  # ragged shards
        a1 = torch.from_numpy(P.fill_normal(P.stream_seed(9, rank), T * shape.d)).cuda()
        a3 = torch.from_numpy(P.fill_normal(P.stream_seed(10, rank), T * shape.d)).cuda()
        uid = broadcast_unique_id()
        ep = ExpertParallelLayer(P.Context(rank), shape, rank, world, 3, uid, max_tokens=1024)
        if dense:
            ep.enable_dense(1024, seed=7)
        res = None
        for _ in range(2):  # twice: epochs and buffer reuse across calls
            res = ep.forward(a1, a3, None, T, renormalize=renorm, dense=dense)
        torch.cuda.synchronize()
        ep.synchronize()
        ref = _single_gpu(P, rank, shape, a1, a3, T, renorm, 1024 if dense else 0)
        ok = all(torch.equal(u, v) for u, v in zip(res, ref))
        m = ep.count_matrix()
        info = dict(out_diff=int((res[0] != ref[0]).sum()), idx_diff=int((res[1] != ref[1]).sum()),
                    matrix=m.tolist())
        ok = ok and int(m[rank].sum()) == int((res[1] < shape.n_ffn).sum())
        ep.close()
        q.put((rank, bool(ok), info))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dense,renorm", [(1, False, False), (2, False, False),
                                                (4, False, False), (2, True, False),
                                                (4, True, False), (2, False, True)])
def test_ep_equals_single_gpu_bitwise(world, dense, renorm):
    port = 29700 + os.getpid() % 100 + 3 * world + 11 * dense + 23 * renorm
    _spawn(_equal_worker, world, port, dense, renorm)


def _empty_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    _init(rank, world, port)
    try:
        import paper_2509_01322_b200 as P
        from paper_2509_01322_b200.ep import ExpertParallelLayer, broadcast_unique_id
        shape = _shape(P)
        T = 0 if rank == world - 1 else 512 + 64 * rank  # the last rank brings no tokens
        a1 = torch.from_numpy(P.fill_normal(P.stream_seed(11, rank), T * shape.d)).cuda()
        a3 = torch.from_numpy(P.fill_normal(P.stream_seed(12, rank), T * shape.d)).cuda()
        ep = ExpertParallelLayer(P.Context(rank), shape, rank, world, 3, broadcast_unique_id(),
                                 max_tokens=1024)
        res = None
        for _ in range(2):
            res = ep.forward(a1.view(T, shape.d), a3.view(T, shape.d), None, T)
        pip = ep.forward_batches([a1] * 3, [a3] * 3, None, T)
        torch.cuda.synchronize()
        ep.synchronize()
        ok = all(torch.equal(u, v) for p in pip for u, v in zip(p, res))
        if T:
            ref = _single_gpu(P, rank, shape, a1, a3, T)
            ok = ok and all(torch.equal(u, v) for u, v in zip(res, ref))
        else:
            ok = ok and all(t.numel() == 0 for t in res)
        # the empty rank still serves its experts: rows arrive from the others
        m = ep.count_matrix()
        ok = ok and int(m[:, world - 1].sum()) > 0 and int(m[world - 1].sum()) == 0
        ep.close()
        q.put((rank, bool(ok), m.tolist()))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ep_rank_without_tokens(world):
    """A rank with an empty shard (T = 0) still exchanges its (zero) counts,
    serves the rows other ranks dispatch to its experts and passes every
    barrier; the other ranks' outputs stay bitwise equal to single-GPU."""
    _spawn(_empty_worker, world, 29900 + os.getpid() % 50 + world)


def _batches_worker(rank, world, port, q, corun):
    import torch
    import torch.distributed as dist
    _init(rank, world, port)
    try:
        import paper_2509_01322_b200 as P
        from paper_2509_01322_b200.ep import ExpertParallelLayer, broadcast_unique_id
        shape = _shape(P)
        T, nb = 704 + 32 * rank, 5
        a1 = [torch.from_numpy(P.fill_normal(P.stream_seed(40 + i, rank), T * shape.d)).cuda()
              for i in range(nb)]
        a3 = [torch.from_numpy(P.fill_normal(P.stream_seed(50 + i, rank), T * shape.d)).cuda()
              for i in range(nb)]
        ep = ExpertParallelLayer(P.Context(rank), shape, rank, world, 3, broadcast_unique_id(),
                                 max_tokens=1024)
        ser = [ep.forward(a1[i], a3[i], None, T) for i in range(nb)]
        pip = ep.forward_batches(a1, a3, None, T, corun_router=corun)
        pip2 = ep.forward_batches(a1[:2], None, None, T)  # again, and without residual
        ser2 = [ep.forward(a1[i], None, None, T)[0] for i in range(2)]
        torch.cuda.synchronize()
        ep.synchronize()
        ok = all(torch.equal(u, v) for s, p in zip(ser, pip) for u, v in zip(s, p))
        ok = ok and all(torch.equal(r, p[0]) for r, p in zip(ser2, pip2))
        ep.close()
        q.put((rank, bool(ok), ""))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,corun", [(1, False), (2, False), (2, True), (4, False)])
def test_ep_pipelined_batches_equal_serial(world, corun):
    """scmoe_ep_layer_forward_batches (front of batch i+1 beside the back of
    batch i, two buffer sets) == serial calls, bit for bit."""
    _spawn(_batches_worker, world, 29820 + os.getpid() % 60 + world + 7 * corun, corun)


def _host_batches_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    _init(rank, world, port)
    try:
        import paper_2509_01322_b200 as P
        from paper_2509_01322_b200.ep import ExpertParallelLayer, broadcast_unique_id
        shape = _shape(P)
        T, nb = 512 + 64 * rank, 3
        a1 = [torch.from_numpy(P.fill_normal(P.stream_seed(70 + i, rank), T * shape.d)
                               .reshape(T, shape.d)).pin_memory() for i in range(nb)]
        a3 = [torch.from_numpy(P.fill_normal(P.stream_seed(80 + i, rank), T * shape.d)
                               .reshape(T, shape.d)).pin_memory() for i in range(nb)]
        ep = ExpertParallelLayer(P.Context(rank), shape, rank, world, 3, broadcast_unique_id(),
                                 max_tokens=1024)
        outs = [torch.empty(T, shape.d).pin_memory() for _ in range(nb)]
        ep.forward_host_batches(a1, a3, outs, None, T)
        torch.cuda.synchronize()
        ok = True
        for i in range(nb):
            ref = ep.forward(a1[i].cuda(), a3[i].cuda(), None, T)[0]
            torch.cuda.synchronize()
            ok = ok and torch.equal(ref.cpu(), outs[i])
        ep.close()
        q.put((rank, bool(ok), ""))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_ep_host_batches_equal_device_calls():
    import torch
    world = min(2, torch.cuda.device_count())
    _spawn(_host_batches_worker, world, 29890 + os.getpid() % 40)


def _controller_worker(rank, world, port, q):
    import numpy as np
    import torch
    import torch.distributed as dist
    _init(rank, world, port)
    try:
        import _oracle as O
        import paper_2509_01322_b200 as P
        from paper_2509_01322_b200.ep import ExpertParallelLayer, broadcast_unique_id
        shape = _shape(P, ke=3)
        T = 512 + 128 * rank
        ep = ExpertParallelLayer(P.Context(rank), shape, rank, world, 3, broadcast_unique_id(),
                                 max_tokens=1024, mu=0.2, mu_decay=0.999)
        E = shape.E
        b = np.zeros(E)
        mu = np.array([0.2])
        ok = True
        for step in range(4):
            a1 = torch.from_numpy(P.fill_normal(P.stream_seed(90 + step, rank), T * shape.d)).cuda()
            out, idx, gates, cnt = ep.forward(a1, None, None, T)
            delta = ep.controller_step(idx, T)
            # one router fed every rank's slots (the reference, router.hpp:144-176)
            parts = [None] * world
            dist.all_gather_object(parts, idx.cpu().numpy().view(np.uint32))
            routed = np.zeros(E, np.uint64)
            seen = np.zeros(1, np.uint64)
            for p_ in parts:
                O.orc().orc_accumulate_counters(O.ptr(p_), p_.size // shape.top_k, shape.top_k,
                                                O.ptr(routed), O.ptr(seen))
            want = np.zeros(E)
            assert O.orc().orc_bias_update(shape.n_ffn, shape.n_zero, shape.top_k,
                                           shape.k_expected, O.ptr(mu), 0.999, O.ptr(b),
                                           O.ptr(routed), O.ptr(seen), O.ptr(want)) == 0
            ok = ok and want.tobytes() == delta.tobytes() and ep.bias().tobytes() == b.tobytes()
        ok = ok and abs(b).sum() > 0
        ep.close()
        q.put((rank, bool(ok), ""))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 4])
def test_ep_controller_global_batch_bitwise(world):
    """the controller sums the per-expert counters and tokens over
    the ranks on the device (ncclAllReduce); every rank's deltas and bias equal
    one router's update over all ranks' slots (oracle), bit for bit."""
    _spawn(_controller_worker, world, 29850 + os.getpid() % 40 + world)


def _torch_worker(rank, world, port, q, transport):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        import paper_2509_01322_b200 as P
        from paper_2509_01322_b200.ep_torch import EPLayer, GpuOps
        shape = _shape(P)
        T = 640 + 64 * rank
        a1 = torch.from_numpy(P.fill_normal(P.stream_seed(9, rank), T * shape.d)).cuda()
        a3 = torch.from_numpy(P.fill_normal(P.stream_seed(10, rank), T * shape.d)).cuda()
        ep = EPLayer(GpuOps(P.Context(rank), shape, rank, world, seed=3), transport=transport)
        res = ep.forward(a1, a3, None, T)
        torch.cuda.synchronize()
        ref = _single_gpu(P, rank, shape, a1, a3, T)
        q.put((rank, all(torch.equal(u, v) for u, v in zip(res, ref)), ""))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, False, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_torch_reference_orchestration_equals_single_gpu(transport):
    """The torch.distributed reference orchestration (ep_torch.py) gives the
    same bits as the single GPU (and hence as the native path)."""
    _spawn(_torch_worker, 2, 29600 + os.getpid() % 40 + (transport == "p2p"), transport)
