"""Measurement probe (not a test): MLA forward value at LongCat widths
(d 6144, d_q 1536, d_kv 512, 64 heads x (128 content + 64 rotary)), exact
fp32 path (csrc/mla.cu), plus cached decode steps.
    python tests/cpp/mla_probe.py [rows] [seq_len] [reps] [--ref THREADS]
Prints one JSON line: device ms per forward, tokens/s, per-stage ms and the
FP32-pipe roofline fraction of each stage (lane-ops = 2 per multiply-add, as
for the router); with --ref, the reference's own mla_block (oracle/_ref) on
one sequence of seq_len rows (token-sharded over sequences is not possible
inside one sequence, so THREADS only matters for several sequences)."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2509_01322_b200 as P  # noqa: E402
from paper_2509_01322_b200.mla import MlaCache, MlaParams, mla_block, mla_infer_step  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
rows = int(args[0]) if len(args) > 0 else 8192
seq = int(args[1]) if len(args) > 1 else 4096
reps = int(args[2]) if len(args) > 2 else 3
d, dq, dkv, H, dhc, dhr = 6144, 1536, 512, 64, 128, 64
ctx = P.Context(0)
# Uniform(variance 1/d) weights, as the bench's synthetic recipe; generated on the device
ws = []
for i, (r, c) in enumerate([(d, dq), (dq, H * dhc), (dq, H * dhr), (d, dkv), (dkv, H * dhc),
                            (dkv, H * dhc), (d, dhr), (H * dhc, d)]):
    t = torch.empty(r * c, dtype=torch.float32, device="cuda")
    ctx._check(P.lib().scmoe_rng_fill_uniform(ctx.handle, P.stream_seed(3, i), 0, r * c, 1.0 / d,
                                              t.data_ptr()))
    ws.append(t.view(r, c))
p = MlaParams(d, dq, dkv, H, dhc, dhr, weights=ws, rope_base=1.0e6,
              precision=int(os.environ.get("MLA_PREC", "0")))  # 1 = tensor-core bf16
h = torch.randn(rows, d, device="cuda")
out = torch.empty(rows, d, device="cuda")
mla_block(h, p, seq, ctx=ctx, out=out)  # warm-up (workspace growth, rope table)
ctx.synchronize()
ctx.profile(True)
ctx.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    mla_block(h, p, seq, ctx=ctx, out=out)
ctx.synchronize()
wall = (time.perf_counter() - t0) / reps * 1e3
prof = {k: v[0] / v[1] for k, v in ctx.profile_flush().items()}
ctx.profile(False)
B = rows // seq
pairs = B * H * seq * (seq + 1) // 2
lane = {
    "mla_proj_h": 2 * rows * d * (dq + dkv + dhr),
    "mla_proj_q": 2 * rows * dq * H * (dhc + dhr),
    "mla_proj_kv": 2 * rows * dkv * 2 * H * dhc,
    "mla_proj_o": 2 * rows * H * dhc * d,
    "mla_scores": 2 * pairs * (dhc + dhr),
    "mla_pv": 2 * pairs * dhc,
}
clk = float(os.environ.get("SM_CLOCK_MHZ", "1965")) * 1e6
peak = 148 * 128 * clk  # FP32 lane-ops/s
stages = {}
for k, ms in prof.items():
    s = {"ms": round(ms, 3)}
    if k in lane:
        s["tlanes_per_s"] = round(lane[k] / (ms * 1e-3) / 1e12, 2)
        s["frac_fp32_pipe"] = round(lane[k] / (ms * 1e-3) / peak, 3)
    stages[k] = s
dev_ms = sum(prof.values())
res = {"probe": "mla_forward", "rows": rows, "seq_len": seq, "widths": [d, dq, dkv, H, dhc, dhr],
       "ms_wall": round(wall, 2), "ms_stages_sum": round(dev_ms, 2),
       "tok_per_s": round(rows / (wall * 1e-3)), "lane_ops_total": sum(lane.values()),
       "frac_fp32_pipe_total": round(sum(lane.values()) / (wall * 1e-3) / peak, 3),
       "stages": stages}
# decode: steps at positions 0..n-1 of one sequence, timed over the last block
n_dec = min(seq, 1024)
cache = MlaCache(p, capacity_hint=n_dec, ctx=ctx)
ht = torch.randn(n_dec, d, device="cuda")
o1 = torch.empty(1, d, device="cuda")
for t in range(n_dec - 32):
    mla_infer_step(p, cache, ht[t:t + 1], t, out=o1)
ctx.synchronize()
t0 = time.perf_counter()
for t in range(n_dec - 32, n_dec):
    mla_infer_step(p, cache, ht[t:t + 1], t, out=o1)
ctx.synchronize()
res["decode_ms_per_step_at_pos"] = [n_dec - 16, round((time.perf_counter() - t0) / 32 * 1e3, 3)]
cache2 = MlaCache(p, capacity_hint=n_dec, ctx=ctx)
for t in range(n_dec - 32):
    mla_infer_step(p, cache2, ht[t:t + 1], t, out=o1)
ctx.synchronize()
ctx.profile(True)
for t in range(n_dec - 32, n_dec):
    mla_infer_step(p, cache2, ht[t:t + 1], t, out=o1)
res["decode_stage_ms"] = {k: round(v[0] / 32, 4) for k, v in ctx.profile_flush().items()}
if "--ref" in sys.argv:
    import _oracle as O
    thr = int(sys.argv[sys.argv.index("--ref") + 1])
    wn = [x.cpu().numpy() for x in ws]
    rs = min(seq, 256)
    hn = h[:rs].cpu().numpy()
    t0 = time.perf_counter()
    rc, _ = O.mla_forward(O.ref(), (d, dq, dkv, H, dhc, dhr), wn, hn, rs, base=1.0e6,
                          threads=thr)
    dt = time.perf_counter() - t0
    res["reference_cpu"] = {"rows": rs, "seq_len": rs, "s": round(dt, 2),
                            "tok_per_s": round(rs / dt, 2), "rc": rc}
print(json.dumps(res))
