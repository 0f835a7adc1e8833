"""Probe which NVLink traffic counters this driver exposes (NVML field values,
nvidia-smi nvlink -gt d) around a known 4 GiB peer copy GPU0 -> GPU1."""
import subprocess
import torch
import pynvml as n

n.nvmlInit()
h = [n.nvmlDeviceGetHandleByIndex(i) for i in range(2)]
F = {k: getattr(n, k) for k in dir(n) if k.startswith("NVML_FI_DEV_NVLINK_THROUGHPUT") or
     k in ("NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES",
           "NVML_FI_DEV_NVLINK_COUNT_XMIT_PACKETS", "NVML_FI_DEV_NVLINK_COUNT_RCV_PACKETS",
           "NVML_FI_DEV_NVLINK_LINK_COUNT")}


def read(dev):
    out = {}
    for name, fid in F.items():
        for scope in [0xFFFFFFFF] + list(range(18)):
            try:
                v = n.nvmlDeviceGetFieldValues(h[dev], [(fid, scope)])[0]
            except Exception as e:
                out[(name, scope)] = f"exc {e}"
                continue
            if v.nvmlReturn == 0:
                out[(name, scope)] = v.value.ullVal
    return out


def smi():
    return subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], capture_output=True,
                          text=True).stdout


a = torch.empty(1 << 31, dtype=torch.int16, device="cuda:0")  # 4 GiB
b = torch.empty_like(a, device="cuda:1")
r0, s0 = read(0), smi()
for _ in range(1):
    b.copy_(a)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
r1, s1 = read(0), smi()
print("NVML field deltas (GPU0, 4 GiB sent):")
for k in sorted(r1, key=str):
    if k in r0 and isinstance(r1[k], int) and isinstance(r0[k], int) and r1[k] != r0[k]:
        print(" ", k, r1[k] - r0[k])
print("supported fields:", sorted({k[0] for k, v in r1.items() if isinstance(v, int)}))
print("nvidia-smi nvlink -gt d before:\n", s0[:1500], "\nafter:\n", s1[:1500])
