"""Measurement probe (not a test): config A (tiny exact fp32 layer, T=512,
d=256, 8+4 experts, top-2, I=128) -- per-stage device time and launch count
of one layer call.  python tests/cpp/config_a_probe.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2509_01322_b200 as P  # noqa: E402
from paper_2509_01322_b200.layer import TINY, DeviceLayer  # noqa: E402

ctx = P.Context(0)
s, T = TINY, 512
lay = DeviceLayer(ctx, s, seed=11)
a1 = torch.randn(T, s.d, device="cuda")
a3 = torch.randn(T, s.d, device="cuda")
idx = torch.empty(T * s.top_k, dtype=torch.int32, device="cuda")
g = torch.empty(T * s.top_k, dtype=torch.float64, device="cuda")
cnt = torch.empty(T, dtype=torch.int32, device="cuda")
out = torch.empty(T, s.d, device="cuda")


def run(n):
    for _ in range(n):
        lay.forward(a1.data_ptr(), a3.data_ptr(), None, T, idx.data_ptr(), g.data_ptr(),
                    cnt.data_ptr(), out.data_ptr())


run(20)
ctx.synchronize()
l0 = ctx.kernel_launches()
ctx.profile(True)
ctx.profile_flush()
run(50)
st = ctx.profile_flush()
ctx.profile(False)
launches = (ctx.kernel_launches() - l0) / 50
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0 = torch.cuda.Stream()
ctx.set_stream(s0.cuda_stream)
with torch.cuda.stream(s0):
    run(20)
    e0.record(s0)
    run(200)
    e1.record(s0)
e1.synchronize()
print(json.dumps({"launches_per_call": launches,
                  "us_per_call": round(e0.elapsed_time(e1) / 200 * 1e3, 2),
                  "stages_us_profiled": {k: round(v[0] / v[1] * 1e3, 2) for k, v in st.items()}}))
