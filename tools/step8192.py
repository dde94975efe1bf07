"""Where the time goes in one configs[4] step (dev tool): device events and host
time per phase of sharding.detect_channel_sharded on all 512 channels."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_15602_b200 as Q
from paper_2510_15602_b200 import sharding
import workloads
with torch.no_grad():
    f, _ = workloads.make_features(1, 8192, seed=1000)
x = f[0].contiguous(); del f; torch.cuda.empty_cache()
cfg = Q.PipelineConfig()
for _ in range(3): sharding.detect_channel_sharded(x, cfg)
torch.cuda.synchronize()
import cProfile, pstats, io
pr = cProfile.Profile()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); e0.record()
pr.enable()
for _ in range(3): sharding.detect_channel_sharded(x, cfg)
pr.disable()
e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
print(json.dumps({"wall_ms": (t1 - t0) / 3 * 1e3, "dev_ms": e0.elapsed_time(e1) / 3}))
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(18); print(s.getvalue()[:3500])
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    sharding.detect_channel_sharded(x, cfg)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14, max_name_column_width=60))
