"""HBM copy bandwidth (torch b.copy_(a), 2 GiB each way) on a rested GPU and right after a burst of
bf16 GEMMs (power-capped clocks): how much of the measured HBM peak any streaming kernel can
expect inside a capped step.   python tools/hbm_hot_probe.py"""
import time

import torch

torch.cuda.set_device(0)
n = 1 << 30
a = torch.empty(n, dtype=torch.bfloat16, device="cuda").normal_()
b = torch.empty_like(a)
x = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
y = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)


def copy_gbs():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    return 2 * n * 2 / (e0.elapsed_time(e1) * 1e-3) / 1e9


copy_gbs()
time.sleep(2)
rested = [copy_gbs() for _ in range(3)]
hot = []
for _ in range(4):
    for _ in range(120):
        torch.matmul(x, y)
    hot.append(copy_gbs())
print("copy GB/s rested:", " ".join(f"{v:.0f}" for v in rested), "| right after 120 bf16 8192^3 GEMMs:",
      " ".join(f"{v:.0f}" for v in hot))
