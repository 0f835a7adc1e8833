"""Measurement probe (not a test): CUPTI timeline of the host tier
(scmoe_layer_forward_host_batches) at the LongCat prefill shape: copies and
kernels of 6 batches, to see where the step loses time against the PCIe
floor.  python tests/cpp/e2e_trace.py"""
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2509_01322_b200 as P  # noqa: E402
from paper_2509_01322_b200.layer import LONGCAT, DeviceLayer  # noqa: E402

T, D, K = 8192, LONGCAT.d, LONGCAT.top_k
ctx = P.Context(0)
lay = DeviceLayer(ctx, LONGCAT, seed=5)


def pinned(shape, dt):
    return torch.empty(shape, dtype=dt).pin_memory().numpy()


hs = []
for i in range(2):
    h = dict(a1=pinned((T, D), torch.float32), a3=pinned((T, D), torch.float32),
             idx=pinned((T * K,), torch.int32), gat=pinned((T * K,), torch.float64),
             cnt=pinned((T,), torch.int32), out=pinned((T, D), torch.float32))
    h["a1"][:] = np.random.default_rng(i).standard_normal((T, D), np.float32)
    h["a3"][:] = 0.5
    hs.append(h)


def host_run(n):
    sl = [hs[i % 2] for i in range(n)]
    lay.forward_host_batches([h["a1"] for h in sl], [h["a3"] for h in sl], None, T,
                             [h["idx"] for h in sl], [h["gat"] for h in sl],
                             [h["cnt"] for h in sl], [h["out"] for h in sl])


host_run(3)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    host_run(6)
    torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if str(e.device_type).endswith("CUDA")),
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    if e.time_range.elapsed_us() > 50:
        print(f"{e.time_range.start - t0:9.0f} {e.time_range.end - t0:9.0f} "
              f"{e.time_range.elapsed_us():8.0f}  {e.name[:70]}")
