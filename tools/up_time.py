import sys, torch
sys.path.insert(0, ".")
import paper_2510_15602_b200 as Q
x = torch.rand(64, 128, 128, dtype=torch.float64, device="cuda")
for _ in range(3): Q.upsample_batch(x, 1024, 1024)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): Q.upsample_batch(x, 1024, 1024)
e1.record(); torch.cuda.synchronize()
print("upsample 64 x 1024^2: %.3f ms" % (e0.elapsed_time(e1) / 20))
