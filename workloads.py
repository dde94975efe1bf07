"""Synthetic benchmark inputs (not product code): seeded stationary textures
with planted square defects, pushed through the reference's default feature
backbone -- Wide-ResNet-50-2 up to block 2 (stride 8, 512 channels) with
random-init weights (torch.manual_seed(0)), ImageNet normalisation -- on the
GPU.  Mirrors the reference's synthetic-data recipe (synth.py kinds noise /
tiles / stripes, planted squares; exporter export.py:71-114) without its
file I/O; there is no network, so no pretrained weights.
"""

from __future__ import annotations

import math

import numpy as np
import torch

_MEAN = (0.485, 0.456, 0.406)
_STD = (0.229, 0.224, 0.225)


def _band_noise(g: torch.Generator, n: int, sigma: float, device) -> torch.Tensor:
    z = torch.randn((n, n), generator=g, device="cpu").to(device)
    f = torch.fft.rfft2(z)
    fy = torch.fft.fftfreq(n, device=device)[:, None]
    fx = torch.fft.rfftfreq(n, device=device)[None, :]
    k = torch.exp(-2 * (math.pi * sigma) ** 2 * (fy ** 2 + fx ** 2))
    out = torch.fft.irfft2(f * k, s=(n, n))
    return out / (out.abs().max() + 1e-12)


def textures(count: int, size: int, seed: int = 0, device="cuda",
             kinds=("noise", "tiles", "stripes"), defect_frac: float = 0.02, n_good: int = 0):
    """(count, 3, size, size) images in [0, 1] and (count, size, size) masks;
    images i < n_good stay clean (no planted square)."""
    g = torch.Generator().manual_seed(seed)
    imgs = torch.empty((count, 3, size, size), device=device)
    masks = torch.zeros((count, size, size), dtype=torch.bool, device=device)
    yy, xx = torch.meshgrid(torch.arange(size, device=device), torch.arange(size, device=device),
                            indexing="ij")
    for i in range(count):
        kind = kinds[i % len(kinds)]
        if kind == "noise":
            base = 0.5 + 0.35 * _band_noise(g, size, 1.5 * size / 256, device)
            img = torch.stack([base, 0.9 * base, 0.8 * base])
        elif kind == "stripes":
            phase = 2.0 * _band_noise(g, size, 4.0 * size / 256, device)
            wave = torch.sin(2 * math.pi * (xx * math.cos(math.pi / 5) + yy * math.sin(math.pi / 5))
                             / (14.0 * size / 256) + phase)
            img = 0.5 + 0.3 * wave + 0.06 * _band_noise(g, size, 0.8 * size / 256, device)
            img = torch.stack([img, 0.95 * img, 0.9 * img])
        else:
            cell = max(1, size // 4)
            mode_b = ((yy // cell + xx // cell) % 2).bool()
            base = 0.5 + 0.3 * _band_noise(g, size, 1.2 * size / 256, device)
            tilt = torch.where(mode_b, 0.06, -0.06)
            img = torch.stack([base + tilt, base, base - tilt])
        side = max(4, int(round(math.sqrt(defect_frac) * size)))
        m = size // 8
        y0 = int(torch.randint(m, size - m - side, (1,), generator=g))
        x0 = int(torch.randint(m, size - m - side, (1,), generator=g))
        if i >= n_good:
            masks[i, y0:y0 + side, x0:x0 + side] = True
            img[:, y0:y0 + side, x0:x0 + side] += 0.28
        imgs[i] = img.clamp(0, 1)
    return imgs, masks


_TRUNK = {}


def backbone(device="cuda"):
    """WRN50-2 conv1..layer2, random init with torch.manual_seed(0) (export.py:71-101)."""
    key = str(device)
    if key not in _TRUNK:
        from torchvision.models import wide_resnet50_2
        torch.manual_seed(0)
        model = wide_resnet50_2(weights=None)
        trunk = torch.nn.Sequential(model.conv1, model.bn1, model.relu, model.maxpool,
                                    model.layer1, model.layer2).eval().to(device)
        _TRUNK[key] = trunk
    return _TRUNK[key]


@torch.no_grad()
def features(images: torch.Tensor, chunk: int = 16) -> torch.Tensor:
    """(B, 3, S, S) images -> (B, 512, S/8, S/8) float32 block-2 features."""
    trunk = backbone(images.device)
    mean = torch.tensor(_MEAN, device=images.device)[:, None, None]
    std = torch.tensor(_STD, device=images.device)[:, None, None]
    outs = []
    prev = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = False
    try:
        for i in range(0, images.shape[0], chunk):
            outs.append(trunk((images[i:i + chunk] - mean) / std).float())
    finally:
        torch.backends.cudnn.allow_tf32 = prev
    return torch.cat(outs).contiguous()


def make_features(count: int, size: int, seed: int = 0, device="cuda"):
    imgs, masks = textures(count, size, seed=seed, device=device)
    return features(imgs), masks
