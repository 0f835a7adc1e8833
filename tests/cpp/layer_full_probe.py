"""Measurement probe (not a test): the full ScMoE layer (model.hpp:355-409) at
LongCat widths -- MLA1 -> dense FFN (12288) -> MLA2, MoE branch (512 + 256
experts, top-12, bf16 tcgen05) -- serial vs overlapped (MoE on its own
stream).  python tests/cpp/layer_full_probe.py [rows] [seq_len] [reps] [mla_precision]
(mla_precision 0 = exact fp32 MLA, 1 = tensor-core bf16 MLA)."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2509_01322_b200 as P  # noqa: E402
from paper_2509_01322_b200.layer import LONGCAT, DenseFFN, DeviceLayer  # noqa: E402
from paper_2509_01322_b200.mla import MlaParams, ScMoELayer  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
seq = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
prec = int(sys.argv[4]) if len(sys.argv) > 4 else 0
d, dq, dkv, H, dhc, dhr = 6144, 1536, 512, 64, 128, 64
ctx = P.Context(0)


def mla(seed):
    ws = []
    for i, (r, c) in enumerate([(d, dq), (dq, H * dhc), (dq, H * dhr), (d, dkv), (dkv, H * dhc),
                                (dkv, H * dhc), (d, dhr), (H * dhc, d)]):
        t = torch.empty(r * c, dtype=torch.float32, device="cuda")
        ctx._check(P.lib().scmoe_rng_fill_uniform(ctx.handle, P.stream_seed(seed, i), 0, r * c,
                                                  1.0 / d, t.data_ptr()))
        ws.append(t.view(r, c))
    return MlaParams(d, dq, dkv, H, dhc, dhr, weights=ws, rope_base=1.0e6, precision=prec)


class _Handle:  # device-initialised router / bank of DeviceLayer
    def __init__(self, h, top_k=None):
        self.h, self.top_k = h, top_k

    def device(self, c):
        return self.h


moe = DeviceLayer(ctx, LONGCAT, seed=1)
layer = ScMoELayer(mla(3), mla(4), DenseFFN(ctx, d, 12288), _Handle(moe.router, LONGCAT.top_k),
                   _Handle(moe.bank), *[torch.ones(d).numpy()] * 4, ctx=ctx)
x = torch.randn(rows, d, device="cuda")
res = {"probe": "scmoe_layer_full", "rows": rows, "seq_len": seq,
       "mla": "tensor-core bf16" if prec else "exact fp32"}
for overlap in (False, True):
    layer.forward(x, seq, overlap=overlap)
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        layer.forward(x, seq, overlap=overlap)
    ctx.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    res["overlap" if overlap else "serial"] = {"ms": round(ms, 2), "tok_per_s": round(rows / ms * 1e3)}
ctx.profile(True)
layer.forward(x, seq, overlap=False)
res["stages_serial_ms"] = {k: round(v[0], 3) for k, v in ctx.profile_flush().items()}
ctx.profile(True)
layer.forward(x, seq, overlap=True)
ctx.profile_flush()
res["timeline_overlap_ms"] = [(n, round(a, 3), round(b, 3)) for n, a, b in ctx.profile_spans()]
print(json.dumps(res))
