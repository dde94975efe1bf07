"""configs[4] per-rank share: 64 channels of one 8192^2 texture (1024^2 feature
plane) through sharding.channel_partial on one GPU (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_15602_b200 as Q
from paper_2510_15602_b200 import sharding, _native as N

c, h, w = int(sys.argv[1]) if len(sys.argv) > 1 else 64, 1024, 1024
g = torch.Generator(device="cuda").manual_seed(0)
base = torch.randn((c, h // 8, w // 8), device="cuda", generator=g)
x = torch.nn.functional.interpolate(base[None], size=(h, w), mode="bilinear")[0]
x = torch.relu(x + 0.1 * torch.randn((c, h, w), device="cuda", generator=g)).contiguous()
cfg = Q.PipelineConfig()
L = N.lib()
ver = L.qfca_score_version(h, w, cfg.n_bins, cfg.patch_size, c, 1, N.PAD_CODES[cfg.pad],
                           cfg.sample_budget, 0)
acc, used = sharding.channel_partial(x, cfg)
torch.cuda.synchronize()
times = []
for _ in range(10):  # per call (each ends in a host sync for the used count)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    acc, used = sharding.channel_partial(x, cfg)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
ms = min(times)
print(json.dumps({"channels": c, "plane": [h, w], "score_version": ver, "ms": round(ms, 2),
                  "ms_per_channel": round(ms / c, 3), "used": used}))
