import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name):
    import numpy as np
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_names(prefix=""):
    # metrics_*.npz / pooling.npz / planted_*.npz belong to test_metrics.py,
    # test_pooling.py and test_planted.py (different layouts)
    return sorted(f[:-4] for f in os.listdir(GOLDEN)
                  if f.endswith(".npz") and f.startswith(prefix)
                  and not f.startswith(("metrics_", "pooling", "planted_")))


def cfg_of(d):
    """PipelineConfig kwargs stored in a golden case."""
    out = {}
    for k, v in d.items():
        if k.startswith("cfg_"):
            v = v.item()
            out[k[4:]] = v
    return out
