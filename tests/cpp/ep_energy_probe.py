"""Energy probe (not a test): dynamic energy per EP layer call on rank 0 --
pipelined batches, serial calls, and serial calls with the row transfers
replaced by no-ops (scmoe_ep_set_comm(0)) -- to locate the expert-parallel
overhead.  Run under torchrun with N GPUs (8192 tokens per GPU)."""
import json
import os
import sys
import time

import pynvml as Nv
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import paper_2509_01322_b200 as P  # noqa: E402
from paper_2509_01322_b200.ep import ExpertParallelLayer, broadcast_unique_id  # noqa: E402
from paper_2509_01322_b200.layer import LONGCAT  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("gloo")
T, D = 8192, LONGCAT.d
ep = ExpertParallelLayer(P.Context(local), LONGCAT, rank, world, 5, broadcast_unique_id(),
                         max_tokens=T)
a1 = torch.from_numpy(P.fill_normal(P.stream_seed(99, rank), T * D, threads=8)).cuda()
a3 = torch.from_numpy(P.fill_normal(P.stream_seed(100, rank), T * D, threads=8)).cuda()
Nv.nvmlInit()
h = Nv.nvmlDeviceGetHandleByIndex(local)
torch.cuda.synchronize()
dist.barrier()
time.sleep(0.3)
e, t = Nv.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
time.sleep(1.0)
idle = (Nv.nvmlDeviceGetTotalEnergyConsumption(h) - e) / 1e3 / (time.perf_counter() - t)


def serial(n):
    for _ in range(n):
        ep.forward(a1, a3, None, T)


def pipelined(n):
    ep.forward_batches([a1] * n, [a3] * n, None, T)


res = {"rank": rank, "world": world, "idle_w": round(idle, 1)}
for name, fn, comm in (("pipelined", pipelined, True), ("serial", serial, True),
                       ("serial_comm_off", serial, False)):
    ep.set_comm(comm)
    fn(10)
    torch.cuda.synchronize()
    dist.barrier()
    n = 200
    e0, w0 = Nv.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    fn(n)
    t1.record()
    t1.synchronize()
    torch.cuda.synchronize()
    time.sleep(0.25)
    e1, w1 = Nv.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
    dist.barrier()
    ms = t0.elapsed_time(t1) / n
    j = ((e1 - e0) / 1e3 - idle * max(0.0, (w1 - w0) - ms * n / 1e3)) / n
    res[name] = {"ms": round(ms, 3), "j_dyn": round(j - idle * ms / 1e3, 3),
                 "avg_w": round(j / ms * 1e3, 1)}
ep.set_comm(True)
if rank == 0:
    print(json.dumps(res), flush=True)
dist.barrier()
ep.close()
dist.destroy_process_group()
