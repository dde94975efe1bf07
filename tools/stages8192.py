"""Dev: per-stage device times of the configs[4] step over 30 steps (which
stage carries the occasional slow steps)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_15602_b200 as Q
from paper_2510_15602_b200 import sharding, _native as N
from paper_2510_15602_b200.quantize import minmax_dev, bins_dev
import workloads
with torch.no_grad():
    feats, _ = workloads.make_features(1, 8192, seed=1000, device=torch.device("cuda"))
x = feats[0].contiguous()
del feats
cfg = Q.PipelineConfig()
c, h, w = x.shape
orig_call = N.call
marks = []


def E():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def call(name, *a):  # mark around the two big kernels
    if name in ("qfca_select_reference",):
        marks.append(("pre-K3", E()))
    r = orig_call(name, *a)
    if name in ("qfca_select_reference",):
        marks.append(("K3", E()))
    return r


N.call = call
L = N.lib()
orig_tiles = L.qfca_score_tiles


for _ in range(3):
    sharding.detect_channel_sharded(x, cfg)
torch.cuda.synchronize()
rows = []
for i in range(30):
    marks.clear()
    e0 = E()
    sharding.detect_channel_sharded(x, cfg)
    e1 = E()
    torch.cuda.synchronize()
    t = {k: e0.elapsed_time(ev) for k, ev in marks}
    tot = e0.elapsed_time(e1)
    rows.append((round(t.get("pre-K3", 0), 2), round(t.get("K3", 0) - t.get("pre-K3", 0), 2),
                 round(tot - t.get("K3", 0), 2), round(tot, 2)))
print("quantize, K3, tiles+finalise, total (ms):")
for r in rows:
    print(r)
