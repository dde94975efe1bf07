import sys, warnings
import torch
sys.path.insert(0, ".")
import paper_2510_15602_b200 as Q
from paper_2510_15602_b200 import sharding
import workloads
with torch.no_grad():
    feats, _ = workloads.make_features(1, 8192, seed=1000, device=torch.device("cuda"))
x = feats[0].contiguous()
del feats
cfg = Q.PipelineConfig()
sharding.detect_channel_sharded(x, cfg)
torch.cuda.synchronize()
torch.cuda.set_sync_debug_mode("warn")
with warnings.catch_warnings(record=True) as w:
    warnings.simplefilter("always")
    sharding.detect_channel_sharded(x, cfg)
    for ww in w: print("SYNC:", str(ww.message)[:200], ww.filename, ww.lineno)
print("done")
