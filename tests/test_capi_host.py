"""CPU-only checks of the C-ABI library and the host logic (no kernels run)."""

import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_functions():
    src = open(os.path.join(ROOT, "include", "qfca_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qfca_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    import ctypes
    from paper_2510_15602_b200 import _native
    lib = ctypes.CDLL(_native.LIB_PATH)
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_native.EXPORTED)


def test_library_is_sm100a():
    import subprocess
    from paper_2510_15602_b200 import _native
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_only_entry_points():
    from paper_2510_15602_b200 import _native as N
    L = N.lib()
    assert L.qfca_abi_version() == 1
    assert L.qfca_sample_stride(64, 64, 4096) == 1
    assert L.qfca_sample_stride(128, 128, 4096) == 2
    assert L.qfca_sample_stride(1024, 1024, 4096) == 16
    from oracle import qfca_oracle as O
    for h, w, b in [(13, 17, 30), (32, 32, 4096), (7, 1000, 100), (1, 1, 1)]:
        assert L.qfca_sample_stride(h, w, b) == O.sample_stride(h, w, b)
    g = L.qfca_score_groups(128, 128, 16, 9, 512, 64, 0, 1, 4096, 0)
    assert 1 <= g <= 512
    import ctypes
    cfg = N.QfcaConfig(16, 9, 1, 4096, 4, 0, 1.0)
    nb = L.qfca_detect_workspace_bytes(64, 512, 64, 64, ctypes.byref(cfg))
    assert nb > 64 * 512 * 64 * 64  # at least the bins
    bad = N.QfcaConfig(16, 8, 1, 4096, 4, 0, 1.0)  # even patch size
    assert L.qfca_detect_workspace_bytes(1, 4, 8, 8, ctypes.byref(bad)) == -1
    zero = N.QfcaConfig(16, 9, 0, 4096, 4, 0, 1.0)  # zero pad: general path only
    assert L.qfca_detect_workspace_bytes(1, 4, 8, 8, ctypes.byref(zero)) == -1
    assert L.qfca_status_str(3).decode().startswith("configuration")


def test_pipeline_config_mirrors_reference():
    from paper_2510_15602_b200 import PipelineConfig, fused_supported
    cfg = PipelineConfig()
    assert (cfg.n_bins, cfg.patch_size, cfg.sigma_s, cfg.reference_mode, cfg.border,
            cfg.sample_budget, cfg.pad) == (16, 9, 1.0, "median-quan", 4, 4096, "reflect")
    assert math.isinf(cfg.sigma_p)
    with pytest.raises(ValueError):
        PipelineConfig(patch_size=4)
    with pytest.raises(ValueError):
        PipelineConfig(n_bins=0)
    with pytest.raises(ValueError):
        PipelineConfig(sigma_s=-1)
    assert fused_supported(cfg)
    assert not fused_supported(PipelineConfig(pad="zero"))
    assert not fused_supported(PipelineConfig(sigma_p=2.0))
    assert not fused_supported(PipelineConfig(reference_mode="quan-mean"))


def test_featuremap_validation():
    from paper_2510_15602_b200 import FeatureMap
    with pytest.raises(ValueError):
        FeatureMap(values=np.zeros((2, 2), np.float32))
    with pytest.raises(ValueError):
        FeatureMap(values=np.zeros((1, 2, 2), np.float32), scale=0)
    with pytest.raises(ValueError):
        FeatureMap(values=np.full((1, 2, 2), np.nan, np.float32))


def test_no_cpu_fallback():
    """Without a GPU, every compute entry point fails loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2510_15602_b200 as Q
    with pytest.raises(RuntimeError, match="CUDA"):
        Q.fit_quantizer(np.zeros((1, 4, 4), np.float32), 4)
    with pytest.raises(RuntimeError, match="CUDA"):
        Q.detect(Q.FeatureMap(values=np.ones((1, 4, 4), np.float32)))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2510_15602_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert "oracle" not in src.replace("oracle/", ""), f
