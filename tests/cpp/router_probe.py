"""Profiling probe (not a test): the router projection alone at the LongCat
prefill shape (T=8192, d=6144, E=768), kernel chosen by SCMOE_ROUTER.
    SCMOE_ROUTER=tma python tests/cpp/router_probe.py [reps]
(SCMOE_PROBE_T=256: the decode batch; SCMOE_SEQ_SMALL picks its tile)
Prints the mean route_topk device time per call."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2509_01322_b200 as P  # noqa: E402
from paper_2509_01322_b200.layer import LONGCAT, DeviceLayer  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ctx = P.Context(0)
layer = DeviceLayer(ctx, LONGCAT, seed=1)
T, d = int(os.environ.get("SCMOE_PROBE_T", "8192")), LONGCAT.d
a1 = torch.randn(T, d, device="cuda")
a3 = torch.randn(T, d, device="cuda")
idx = torch.empty(T * LONGCAT.top_k, dtype=torch.int32, device="cuda")
gates = torch.empty(T * LONGCAT.top_k, dtype=torch.float64, device="cuda")
cnt = torch.empty(T, dtype=torch.int32, device="cuda")
out = torch.empty(T, d, device="cuda")
for _ in range(3):  # warm-up (workspace growth, first launches)
    layer.forward(a1.data_ptr(), a3.data_ptr(), None, T, idx.data_ptr(), gates.data_ptr(),
                  cnt.data_ptr(), out.data_ptr())
ctx.synchronize()
ctx.profile(True)
for _ in range(reps):
    layer.forward(a1.data_ptr(), a3.data_ptr(), None, T, idx.data_ptr(), gates.data_ptr(),
                  cnt.data_ptr(), out.data_ptr())
ctx.synchronize()
prof = ctx.profile_flush()
print(os.environ.get("SCMOE_ROUTER", "auto"), "T", T, "small", os.environ.get("SCMOE_SEQ_SMALL", "16"), {k: round(v[0] / v[1], 4) for k, v in prof.items()})
