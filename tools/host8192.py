"""Host-side time per C-ABI call in one configs[4] step (dev tool)."""
import os, sys, time, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_15602_b200 as Q
from paper_2510_15602_b200 import sharding, _native as N
import workloads
with torch.no_grad():
    f, _ = workloads.make_features(1, 8192, seed=1000)
x = f[0].contiguous(); del f; torch.cuda.empty_cache()
cfg = Q.PipelineConfig()
for _ in range(3): sharding.detect_channel_sharded(x, cfg)
torch.cuda.synchronize()
acc = collections.defaultdict(float)
orig = N.call
def timed(name, *a):
    t0 = time.perf_counter(); orig(name, *a); acc[name] += time.perf_counter() - t0
N.call = timed
for _ in range(5):
    t0 = time.perf_counter()
    sharding.detect_channel_sharded(x, cfg)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print("step wall ms", round((time.perf_counter() - t0) * 1e3, 2), "host until return", round((t1 - t0) * 1e3, 2))
print({k: round(v / 5 * 1e3, 3) for k, v in sorted(acc.items(), key=lambda kv: -kv[1])})
