"""Which NVLink byte counters does this box expose?  Prints nvidia-smi nvlink
sub-commands' output and NVML field values (TX/RX data throughput) for GPU 0
before and after a 1 GiB peer copy GPU0 -> GPU1."""
import subprocess

import pynvml
import torch


def smi(*args):
    r = subprocess.run(["nvidia-smi", *args], capture_output=True, text=True, timeout=60)
    return (r.stdout + r.stderr)[:3000]


def nvml(h):
    out = {}
    for name in ("NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX",
                 "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX"):
        fid = getattr(pynvml, name, None)
        if fid is None:
            continue
        for scope in (0, 0xFFFFFFFF):
            try:
                v = pynvml.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
                out[f"{name}@{scope}"] = (v.nvmlReturn, v.value.ullVal)
            except Exception as e:  # noqa: BLE001
                out[f"{name}@{scope}"] = repr(e)[:80]
    return out


print(smi("nvlink", "-h")[:1500])
print(smi("nvlink", "-s", "-i", "0")[:1500])
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
print("before", nvml(h))
print(smi("nvlink", "-gt", "d", "-i", "0")[:1500])
a = torch.ones(1 << 28, device="cuda:0")
b = torch.empty(1 << 28, device="cuda:1")
for _ in range(4):
    b.copy_(a)
torch.cuda.synchronize()
print("after 4 GiB", nvml(h))
print(smi("nvlink", "-gt", "d", "-i", "0")[:1500])
