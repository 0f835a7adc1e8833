"""Profiling probe (not a test): the layer at an expert-parallel shard shape on
one GPU -- n_ffn local experts, T tokens, so tokens per expert ~ T*8/n_ffn
(EP4 LongCat: n_ffn=128, T=8192 -> ~512).
    python tests/cpp/gemm_probe.py [n_ffn] [T] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2509_01322_b200 as P  # noqa: E402
from paper_2509_01322_b200.layer import DeviceLayer, LayerShape  # noqa: E402

n_ffn = int(sys.argv[1]) if len(sys.argv) > 1 else 128
T = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
shape = LayerShape(d=6144, n_ffn=n_ffn, n_zero=n_ffn // 2, top_k=12, k_expected=8, inter=2048)
ctx = P.Context(0)
layer = DeviceLayer(ctx, shape, seed=1)
a1 = torch.randn(T, shape.d, device="cuda")
a3 = torch.randn(T, shape.d, device="cuda")
idx = torch.empty(T * 12, dtype=torch.int32, device="cuda")
gates = torch.empty(T * 12, dtype=torch.float64, device="cuda")
cnt = torch.empty(T, dtype=torch.int32, device="cuda")
out = torch.empty(T, shape.d, device="cuda")
run = lambda: layer.forward(a1.data_ptr(), a3.data_ptr(), None, T, idx.data_ptr(),  # noqa: E731
                            gates.data_ptr(), cnt.data_ptr(), out.data_ptr())
run()
ctx.synchronize()
ctx.profile(True)
for _ in range(reps):
    run()
ctx.synchronize()
prof = ctx.profile_flush()
slots = int((idx.cpu() < n_ffn).sum())
g = prof["gemm1_tcgen05"][0] / reps + prof["gemm2_tcgen05"][0] / reps
print(f"n_ffn={n_ffn} T={T} slots={slots} tok/expert={slots / n_ffn:.0f} "
      f"gemm {g:.3f} ms = {4.0 * slots * 6144 * 2048 / (g / 1e3) / 1e12:.0f} TFLOP/s",
      {k: round(v[0] / v[1], 4) for k, v in prof.items()})
