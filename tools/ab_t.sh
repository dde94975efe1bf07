#!/bin/bash
# A/B of detect_batch time per 1024^2 image at one patch size (dev): bash tools/ab_t.sh <lib_a> <T> [reps]
A=$1; T=$2; N=${3:-2}
for i in $(seq $N); do
  for L in "$A" ""; do
    QFCA_B200_LIB=$L python - $T <<'PY'
import os, sys, torch
sys.path.insert(0, ".")
import paper_2510_15602_b200 as Q
import workloads
t = int(sys.argv[1])
x, _ = workloads.make_features(8, 1024, seed=7)
cfg = Q.PipelineConfig(patch_size=t)
for _ in range(2): Q.detect_batch(x, cfg)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): Q.detect_batch(x, cfg)
e1.record(); torch.cuda.synchronize()
print(os.environ.get("QFCA_B200_LIB", "") .split("/")[-1] or "default", t, round(e0.elapsed_time(e1) / 5 / 8, 4), "ms/image")
PY
  done
done
