"""Energy probe (not a test): dynamic energy per layer call of the MoE back
half at an expert-parallel shard shape (n_ffn local experts, T tokens) --
does an expert whose rows spill into a second token tile (its weight block
streamed through L2 -> shared memory twice) cost more joules per token?
    python tests/cpp/gemm_energy_probe.py n_ffn T1 [T2 ...]"""
import json
import os
import sys
import time

import pynvml as N
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2509_01322_b200 as P  # noqa: E402
from paper_2509_01322_b200.layer import DeviceLayer, LayerShape  # noqa: E402

n_ffn = int(sys.argv[1])
Ts = [int(t) for t in sys.argv[2:]]
N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)
shape = LayerShape(d=6144, n_ffn=n_ffn, n_zero=n_ffn // 2, top_k=12, k_expected=8, inter=2048)
ctx = P.Context(0)
layer = DeviceLayer(ctx, shape, seed=1)
torch.cuda.synchronize()
time.sleep(0.3)
e, t = N.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
time.sleep(1.0)
idle = (N.nvmlDeviceGetTotalEnergyConsumption(h) - e) / 1e3 / (time.perf_counter() - t)
out = {"idle_w": round(idle, 1), "n_ffn": n_ffn}
for T in Ts:
    a1 = torch.randn(T, shape.d, device="cuda")
    a3 = torch.randn(T, shape.d, device="cuda")
    idx = torch.empty(T * 12, dtype=torch.int32, device="cuda")
    gates = torch.empty(T * 12, dtype=torch.float64, device="cuda")
    cnt = torch.empty(T, dtype=torch.int32, device="cuda")
    o = torch.empty(T, shape.d, device="cuda")
    hmoe = torch.empty(T, shape.d, device="cuda")
    hb = torch.empty(T, shape.d, dtype=torch.bfloat16, device="cuda")
    ctx._check(P.lib().scmoe_rmsnorm_route(ctx.handle, layer.router, a1.data_ptr(), None, T,
                                           hmoe.data_ptr(), hb.data_ptr(), idx.data_ptr(),
                                           gates.data_ptr(), cnt.data_ptr()))

    def back(n):
        for _ in range(n):
            ctx._check(P.lib().scmoe_moe_forward(ctx.handle, layer.bank, hmoe.data_ptr(), T,
                                                 idx.data_ptr(), gates.data_ptr(), 12,
                                                 n_ffn // 2, 0, a3.data_ptr(), o.data_ptr()))
    back(20)
    torch.cuda.synchronize()
    n = 300
    e0, w0 = N.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    back(n)
    t1.record()
    t1.synchronize()
    time.sleep(0.25)
    e1, w1 = N.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
    ms = t0.elapsed_time(t1) / n
    j = ((e1 - e0) / 1e3 - idle * max(0.0, (w1 - w0) - ms * n / 1e3)) / n
    slots = int((idx < n_ffn).sum())
    out[T] = {"tok_per_expert": round(slots / n_ffn, 1), "ms": round(ms, 3),
              "j_dyn": round(j - idle * ms / 1e3, 3),
              "mj_dyn_per_kslot": round((j - idle * ms / 1e3) / slots * 1e6, 3)}
print(json.dumps(out))
