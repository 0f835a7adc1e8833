"""Debug probe (not a test): run the tensor-core MLA forward on one shape and
print rel-L2 vs the exact device path.  python tests/cpp/mla_tc_shapes.py
d dq dkv H dhc dhr seq nseq"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2509_01322_b200 as P  # noqa: E402
from paper_2509_01322_b200.mla import MlaParams, mla_block  # noqa: E402

d, dq, dkv, H, dhc, dhr, seq, nseq = map(int, sys.argv[1:9])
ctx = P.Context(0)
ws = []
for i, (r, c) in enumerate([(d, dq), (dq, H * dhc), (dq, H * dhr), (d, dkv), (dkv, H * dhc),
                            (dkv, H * dhc), (d, dhr), (H * dhc, d)]):
    t = torch.empty(r * c, dtype=torch.float32, device="cuda")
    ctx._check(P.lib().scmoe_rng_fill_uniform(ctx.handle, P.stream_seed(3, i), 0, r * c, 1.0 / d,
                                              t.data_ptr()))
    ws.append(t.view(r, c))
h = torch.randn(seq * nseq, d, device="cuda")
outs = []
for prec in (0, 1):
    p = MlaParams(d, dq, dkv, H, dhc, dhr, weights=ws, rope_base=1.0e6, precision=prec)
    o = torch.empty(seq * nseq, d, device="cuda")
    mla_block(h, p, seq, ctx=ctx, out=o)
    ctx.synchronize()
    outs.append(o.double())
err = float(((outs[1] - outs[0]).norm() / outs[0].norm()).item())
print(f"shape {sys.argv[1:9]}: rel-L2 {err:.3e}", flush=True)
