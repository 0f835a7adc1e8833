"""Measurement probe (not a test): dynamic energy of the N=1 layer's parts at
the LongCat shape -- the decode step (256 tokens: the expert weights streamed
from HBM with almost no tensor work), the prefill back half (8192 tokens:
same weights + 3.3 TFLOP), the exact router alone -- from NVML's energy
counter, minus idle power x time.  Splits the prefill's joules into weight
streaming vs tensor work vs the FP32 router.
    python tests/cpp/energy_split_probe.py"""
import json
import os
import sys
import time

import pynvml as N
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import corun_probe as cp  # noqa: E402  (layer + schedules at T = 8192)

N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)
lay, T = cp.layer, cp.T
Tc = 256
dev = dict(idx=torch.empty(Tc * 12, dtype=torch.int32, device="cuda"),
           gates=torch.empty(Tc * 12, dtype=torch.float64, device="cuda"),
           cnt=torch.empty(Tc, dtype=torch.int32, device="cuda"),
           out=torch.empty(Tc, 6144, device="cuda"))


def decode(n):
    for i in range(n):
        off = (i % (T // Tc)) * Tc * 6144 * 4
        lay.forward(cp.a1.data_ptr() + off, cp.a3.data_ptr() + off, None, Tc,
                    dev["idx"].data_ptr(), dev["gates"].data_ptr(), dev["cnt"].data_ptr(),
                    dev["out"].data_ptr())


def measure(fn, n):
    fn(max(2, n // 4))
    torch.cuda.synchronize()
    e0, w0 = N.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(cp.stream)
    fn(n)
    t1.record(cp.stream)
    t1.synchronize()
    time.sleep(0.25)
    e1, w1 = N.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
    ms = t0.elapsed_time(t1) / n
    return ms, (e1 - e0) / 1e3, (w1 - w0)


torch.cuda.synchronize()
time.sleep(0.3)
e, t = N.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
time.sleep(1.0)
idle = (N.nvmlDeviceGetTotalEnergyConsumption(h) - e) / 1e3 / (time.perf_counter() - t)
res = {"idle_w": round(idle, 1)}
with torch.cuda.stream(cp.stream):
    # the router first: the back half consumes the routing it writes
    for name, fn, n in (("router_8192", lambda k: (setattr(cp, "n", k), cp.router_only()), 300),
                        ("moe_back_8192", lambda k: (setattr(cp, "n", k), cp.moe_only()), 250),
                        ("decode_256", decode, 400),
                        ("pipelined_8192", lambda k: (setattr(cp, "n", k), cp.pipelined()), 250)):
        ms, j, wall = measure(fn, n)
        busy = ms * n / 1e3
        e_total = (j - idle * max(0.0, wall - busy)) / n  # idle energy outside the busy window removed
        res[name] = {"ms": round(ms, 3), "j_per_call": round(e_total, 3),
                     "j_dynamic": round(e_total - idle * ms / 1e3, 3),
                     "avg_w": round(e_total / ms * 1e3, 1)}
print(json.dumps(res))
