"""Measurement probe (not a test): energy per batch of the N=1 headline
workload (LongCat prefill, 8192 tokens) for the router alone, the MoE GEMM
branch alone, both serially, and both co-resident (the pipelined schedule
bench.py times).  NVML's total-energy counter (mJ) is read around N batches,
so J/batch is exact over the run; with the enforced power limit it gives
the power-bound floor of a schedule:  ms >= J_per_batch / P_limit.

    python tests/cpp/power_probe.py [batches]"""
import json
import os
import sys
import threading
import time

import pynvml as N
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import corun_probe as cp  # noqa: E402  (builds the layer and the four schedules)

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 40
N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)
limit_w = N.nvmlDeviceGetEnforcedPowerLimit(h) / 1e3
out = {"probe": "power", "batches": nb, "tokens_per_batch": cp.T, "power_limit_w": limit_w,
       "sm_max_mhz": N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM), "modes": {}}


def sample(stop, clocks, watts):
    while not stop.is_set():
        clocks.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
        watts.append(N.nvmlDeviceGetPowerUsage(h) / 1e3)
        time.sleep(0.005)


cp.n = nb
torch.cuda.synchronize()
time.sleep(0.3)
mj, t = N.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
time.sleep(1.0)
idle_w = (N.nvmlDeviceGetTotalEnergyConsumption(h) - mj) / 1e3 / (time.perf_counter() - t)
out["idle_w"] = round(idle_w, 1)
with torch.cuda.stream(cp.stream):
    for name, fn in (("router_only", cp.router_only), ("moe_only", cp.moe_only),
                     ("serial", cp.serial), ("pipelined", cp.pipelined)):
        fn()  # warm: the same mode for as long as the measured run
        torch.cuda.synchronize()
        clocks, watts, stop = [], [], threading.Event()
        th = threading.Thread(target=sample, args=(stop, clocks, watts))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        mj0, w0 = N.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
        th.start()
        e0.record(cp.stream)
        fn()
        e1.record(cp.stream)
        e1.synchronize()
        stop.set()
        th.join()
        time.sleep(0.2)  # the energy counter lags the load
        mj1, w1 = N.nvmlDeviceGetTotalEnergyConsumption(h), time.perf_counter()
        ms = e0.elapsed_time(e1) / nb
        idle_s = max(0.0, (w1 - w0) - ms * nb / 1e3)  # wall time the GPU sat idle
        j = ((mj1 - mj0) / 1e3 - idle_w * idle_s) / nb
        clocks.sort()
        watts.sort()
        out["modes"][name] = {
            "ms_per_batch": round(ms, 3), "j_per_batch": round(j, 3),
            "avg_w": round(j / ms * 1e3, 1),
            "sm_mhz_median": clocks[len(clocks) // 2] if clocks else None,
            "power_w_median": watts[len(watts) // 2] if watts else None,
            "power_floor_ms": round(j / limit_w * 1e3, 3)}
print(json.dumps(out))
