"""Dev: time quantize_dev (K1+K2 fused) on configs[2] / configs[1]-shaped planes."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2510_15602_b200 import quantize
for (planes, hw) in ((64 * 512, 128 * 128), (64 * 512, 64 * 64)):
    x = torch.rand(planes, hw, device="cuda") * 3.0
    for _ in range(3):
        r = quantize.quantize_dev(x, planes, hw, 16)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        r = quantize.quantize_dev(x, planes, hw, 16)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    gb = planes * hw * 5 / 1e9
    print(f"planes {planes} x {hw}: {ms:.3f} ms, {gb / ms:.2f} TB/s")
