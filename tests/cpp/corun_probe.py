"""Profiling probe (not a test): the N=1 headline workload (LongCat prefill,
8192 tokens) as ncu RANGES, so concurrent kernels are measured together:

    range 1: 4 pipelined batches (scmoe_layer_forward_batches: the co-resident
             router beside the grouped GEMMs -- what bench.py times)
    range 2: 4 serial batches (scmoe_layer_forward: no co-residency)

    ncu --replay-mode app-range --profile-from-start off --metrics ... \
        python tests/cpp/corun_probe.py

Without ncu it prints the event-timed ms per batch of both schedules."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2509_01322_b200 as P  # noqa: E402
from paper_2509_01322_b200.layer import LONGCAT, DeviceLayer  # noqa: E402

T, n = 8192, int(os.environ.get("PROBE_BATCHES", "4"))
REPS = int(os.environ.get("PROBE_REPS", "1"))
ctx = P.Context(0)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)
layer = DeviceLayer(ctx, LONGCAT, seed=5)
a1 = torch.from_numpy(P.fill_normal(P.stream_seed(99, 0), T * LONGCAT.d, threads=16)).cuda()
a3 = torch.from_numpy(P.fill_normal(P.stream_seed(100, 0), T * LONGCAT.d, threads=16)).cuda()
sets = [dict(idx=torch.empty(T * 12, dtype=torch.int32, device="cuda"),
             gates=torch.empty(T * 12, dtype=torch.float64, device="cuda"),
             cnt=torch.empty(T, dtype=torch.int32, device="cuda"),
             out=torch.empty(T, LONGCAT.d, device="cuda")) for _ in range(2)]


def pipelined():
    sel = [sets[i & 1] for i in range(n)]
    layer.forward_batches([a1.data_ptr()] * n, [a3.data_ptr()] * n, None, T,
                          [b["idx"].data_ptr() for b in sel], [b["gates"].data_ptr() for b in sel],
                          [b["cnt"].data_ptr() for b in sel], [b["out"].data_ptr() for b in sel])


hmoe = torch.empty(T, LONGCAT.d, device="cuda")
hb = torch.empty(T, LONGCAT.d, dtype=torch.bfloat16, device="cuda")


def router_only():
    """rmsnorm + the co-resident router kernel + top-K, alone (n batches)."""
    ctx.set_overlapped(True)
    for i in range(n):
        b = sets[i & 1]
        ctx._check(P.lib().scmoe_rmsnorm_route(ctx.handle, layer.router, a1.data_ptr(), None, T,
                                               hmoe.data_ptr(), hb.data_ptr(), b["idx"].data_ptr(),
                                               b["gates"].data_ptr(), b["cnt"].data_ptr()))
    ctx.set_overlapped(False)


def moe_only():
    """permute + gather + the two grouped GEMMs + combine, alone (n batches)."""
    for i in range(n):
        b = sets[0]
        ctx._check(P.lib().scmoe_moe_forward(ctx.handle, layer.bank, hmoe.data_ptr(), T,
                                             b["idx"].data_ptr(), b["gates"].data_ptr(), 12, 256, 0,
                                             a3.data_ptr(), b["out"].data_ptr()))


def serial():
    for i in range(n):
        b = sets[i & 1]
        layer.forward(a1.data_ptr(), a3.data_ptr(), None, T, b["idx"].data_ptr(),
                      b["gates"].data_ptr(), b["cnt"].data_ptr(), b["out"].data_ptr())


if __name__ == "__main__":  # power_probe.py imports the schedules only
    with torch.cuda.stream(stream):
        pipelined()
        serial()
        ctx.synchronize()
        router_only()
        moe_only()
        ctx.synchronize()
        best = {}
        for rep in range(REPS):
            for name, fn in (("pipelined", pipelined), ("serial", serial), ("router_only", router_only),
                             ("moe_only", moe_only)):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                torch.cuda.profiler.start()
                e0.record(stream)
                fn()
                e1.record(stream)
                e1.synchronize()
                torch.cuda.synchronize()
                torch.cuda.profiler.stop()
                ms = e0.elapsed_time(e1) / n
                best[name] = min(best.get(name, 1e9), ms)
        for name, ms in best.items():
            print(f"{name}: {ms:.3f} ms per batch" + (f" (min of {REPS})" if REPS > 1 else ""),
                  flush=True)
        if os.environ.get("PROBE_STAGES"):
            for name, fn in (("pipelined", pipelined), ("serial", serial)):
                ctx.profile(True)
                ctx.profile_flush()
                fn()
                st = ctx.profile_flush()
                ctx.profile(False)
                print(name, {k: round(v[0] / v[1], 3) for k, v in st.items()}, flush=True)
