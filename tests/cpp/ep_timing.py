"""Diagnostic (not a test): EP layer step time for blocking vs async
collectives and chunk counts.  torchrun --nproc-per-node N tests/cpp/ep_timing.py"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    import paper_2509_01322_b200 as P
    from paper_2509_01322_b200.ep_torch import EPLayer, GpuOps
    from paper_2509_01322_b200.layer import LONGCAT
    T, D = 8192, LONGCAT.d
    ctx = P.Context(rank)
    ops = GpuOps(ctx, LONGCAT, rank, world, seed=5)
    a1 = torch.from_numpy(P.fill_normal(P.stream_seed(99, rank), T * D, threads=16)).cuda()
    a3 = torch.from_numpy(P.fill_normal(P.stream_seed(100, rank), T * D, threads=16)).cuda()
    for async_comm in (False, True):
        for chunks in (1, 2):
            ep = EPLayer(ops, async_comm=async_comm)
            for _ in range(2):
                ep.forward(a1, a3, None, T, chunks=chunks)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                ep.forward(a1, a3, None, T, chunks=chunks)
            e1.record()
            e1.synchronize()
            ms = torch.tensor([e0.elapsed_time(e1) / 5], device="cuda")
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            if rank == 0:
                print(f"world={world} async={async_comm} chunks={chunks}: {ms.item():.3f} ms",
                      flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
