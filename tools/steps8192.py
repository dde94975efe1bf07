"""Dev: per-step device times of the configs[4] step (distribution)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_15602_b200 as Q
from paper_2510_15602_b200 import sharding
import workloads
with torch.no_grad():
    feats, _ = workloads.make_features(1, 8192, seed=1000, device=torch.device("cuda"))
x = feats[0].contiguous()
del feats
torch.cuda.empty_cache()
cfg = Q.PipelineConfig()
for _ in range(3):
    sharding.detect_channel_sharded(x, cfg)
torch.cuda.synchronize()
ts = []
for i in range(30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sharding.detect_channel_sharded(x, cfg)
    e1.record()
    torch.cuda.synchronize()
    ts.append(round(e0.elapsed_time(e1), 2))
print(ts)
