"""Measurement probe (not a test): the launch list of an expert-parallel
step, captured by CUPTI through torch.profiler (the image has no nsys).  Run
under torchrun with N GPUs:

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tests/cpp/ep_trace.py OUT_PREFIX

Each rank traces 4 pipelined layer calls (scmoe_ep_layer_forward_batches,
8192 tokens per GPU, the bench's headline EP schedule) plus one
controller step, and writes OUT_PREFIX_rank{r}.json: every GPU kernel in the
region (name, count, total device us), the CUDA runtime / driver calls made
in it, and the host-synchronising ones among them -- the evidence that the
N>1 region launches only this repo's kernels (and NCCL's for the controller
all-reduce) with no host synchronisation per batch."""
import json
import os
import sys
from collections import defaultdict

import torch
import torch.distributed as dist
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import paper_2509_01322_b200 as P  # noqa: E402
from paper_2509_01322_b200.ep import ExpertParallelLayer, broadcast_unique_id  # noqa: E402
from paper_2509_01322_b200.layer import LONGCAT  # noqa: E402

prefix = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ep_trace"
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
dist.init_process_group("gloo")
T, D, NB = 8192, LONGCAT.d, 4
ctx = P.Context(torch.cuda.current_device())
ep = ExpertParallelLayer(ctx, LONGCAT, rank, world, 5, broadcast_unique_id(), max_tokens=T,
                         mu=0.2, mu_decay=0.999)
a1 = torch.from_numpy(P.fill_normal(P.stream_seed(99, rank), T * D, threads=8)).cuda()
a3 = torch.from_numpy(P.fill_normal(P.stream_seed(100, rank), T * D, threads=8)).cuda()
for _ in range(2):
    res = ep.forward_batches([a1] * NB, [a3] * NB, None, T)
    ep.controller_step(res[-1][1], T, update=True, want_delta=False)
torch.cuda.synchronize()
dist.barrier()
launches0 = ep.kernel_launches()
CORUN = bool(int(os.environ.get("EP_CORUN", "0")))  # the co-resident router variant
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    res = ep.forward_batches([a1] * NB, [a3] * NB, None, T, corun_router=CORUN)
    ep.controller_step(res[-1][1], T, update=True, want_delta=False)
    torch.cuda.synchronize()
launches = ep.kernel_launches() - launches0

kern = defaultdict(lambda: [0, 0.0])
api = defaultdict(int)
for e in prof.events():
    dt = str(e.device_type)
    if dt.endswith("CUDA"):
        kern[e.name][0] += 1
        kern[e.name][1] += e.device_time_total if hasattr(e, "device_time_total") else 0.0
    elif e.name.startswith(("cuda", "cu")) and not e.name.startswith("cudaGetDevice"):
        api[e.name] += 1
# host-blocking calls (cudaMemcpyAsync here is the device-to-device copy of
# the per-batch plan, asynchronous); each with its start relative to the
# last kernel launch call of the region: > 0 = issued after every launch
launch_api = ("cudaLaunchKernel", "cuLaunchKernelEx", "cuLaunchKernel", "cudaLaunchKernelExC")
cpu_ev = sorted((e for e in prof.events() if not str(e.device_type).endswith("CUDA")),
                key=lambda e: e.time_range.start)
last_launch = max((e.time_range.start for e in cpu_ev if e.name in launch_api), default=0)
syncs = [{"call": e.name, "start_us_after_last_launch": round(e.time_range.start - last_launch, 1),
          "dur_us": round(e.time_range.elapsed_us(), 1)}
         for e in cpu_ev if "Synchronize" in e.name or e.name in ("cudaMemcpy", "cuMemcpyDtoH")]
in_region = [x for x in syncs if x["start_us_after_last_launch"] < 0]
copies = {k: kern.pop(k)[0] for k in [k for k in kern if k.startswith(("Memcpy", "Memset"))]}
own = {k: v for k, v in kern.items() if not k.lower().startswith("nccl")}
out = {"rank": rank, "world": world, "region": f"{NB} pipelined EP layer calls "
       f"({T} tokens per GPU) + 1 controller step, then one torch.cuda.synchronize()",
       "kernel_launches_counted_by_library": launches,
       "gpu_kernels": {k: {"count": v[0], "device_us": round(v[1], 1)}
                       for k, v in sorted(kern.items(), key=lambda kv: -kv[1][1])},
       "n_kernel_launches_traced": sum(v[0] for v in kern.values()),
       "n_repo_kernel_launches": sum(v[0] for v in own.values()),
       "n_nccl_kernel_launches": sum(v[0] for v in kern.values()) - sum(v[0] for v in own.values()),
       "device_copies": copies,
       "runtime_api_calls": dict(sorted(api.items())),
       "host_synchronising_calls": syncs,
       "host_syncs_between_launches": len(in_region),
       "note": "expected: one cudaDeviceSynchronize after the last launch (the region's "
               "closing torch.cuda.synchronize(), possibly another from the profiler "
               "exit) and none between launches: the library issues no host "
               "synchronisation per batch or per controller step"}
os.makedirs(os.path.dirname(prefix) or ".", exist_ok=True)
with open(f"{prefix}_rank{rank}.json", "w") as f:
    json.dump(out, f, indent=1)
if rank == 0:
    prof.export_chrome_trace(f"{prefix}_rank0.trace.json")
    # device timeline of the region (kernel, stream, start/end us from the first kernel)
    ks = sorted((e for e in prof.events() if str(e.device_type).endswith("CUDA")),
                key=lambda e: e.time_range.start)
    if ks:
        t0 = ks[0].time_range.start
        with open(f"{prefix}_rank0.timeline.txt", "w") as f:
            for e in ks:
                f.write(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f} "
                        f"{e.time_range.elapsed_us():8.1f}  {e.name[:90]}\n")
print(json.dumps({k: out[k] for k in ("rank", "n_kernel_launches_traced", "n_repo_kernel_launches",
                                      "n_nccl_kernel_launches", "host_syncs_between_launches",
                                      "kernel_launches_counted_by_library")}), flush=True)
dist.barrier()
ep.close()
dist.destroy_process_group()
