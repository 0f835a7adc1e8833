import sys

import torch
sys.path.insert(0, '.')
import bench
x = torch.randn(8192, 8192, device='cuda')
with bench.ClockSampler(0) as c:
    for _ in range(200): y = x @ x
    torch.cuda.synchronize()
print(c.summary())
import pynvml as n
n.nvmlInit(); h = n.nvmlDeviceGetHandleByIndex(0)
print(n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM), n.nvmlDeviceGetPowerUsage(h), n.nvmlDeviceGetCurrentClocksEventReasons(h))
