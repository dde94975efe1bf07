"""Feature backbone on the GPU (reference exporter, export.py:71-143).

The reference exports features with a Wide-ResNet-50-2 trunk (conv1 .. layer2,
stride 8, 512 channels) on the CPU, one image at a time: PIL bilinear resize,
ImageNet normalisation, ``trunk(x)``, QTF1 file.  Here the same trunk runs on
the GPU in batches (cuDNN convolutions, TF32 off so the features are fp32
like the reference's) and the features stay resident for ``detect_batch``:
the step before the scoring path without a host round trip.  Weights:
"random" (torch.manual_seed(0), the reference's default for tests and the
bench), "pretrained" needs torchvision's cache (no network here), or a .pth
path.
"""

from __future__ import annotations

import os

import torch

MEAN = (0.485, 0.456, 0.406)
STD = (0.229, 0.224, 0.225)
STRIDE = 8

__all__ = ["WeightsError", "build_backbone", "normalize", "extract_features", "STRIDE"]


class WeightsError(Exception):
    """export.py WeightsError: weights could not be obtained."""


def build_backbone(weights: str = "random", device=None) -> torch.nn.Module:
    """export.py:71-101: WRN50-2 stem + layer1 + layer2, eval mode, on the GPU."""
    from torchvision.models import wide_resnet50_2
    if weights == "random":
        torch.manual_seed(0)
        model = wide_resnet50_2(weights=None)
    elif weights == "pretrained":
        try:
            from torchvision.models import Wide_ResNet50_2_Weights
            model = wide_resnet50_2(weights=Wide_ResNet50_2_Weights.IMAGENET1K_V1)
        except Exception as e:  # no cached weights and no network
            raise WeightsError("could not obtain pretrained weights; pass a .pth path") from e
    else:
        if not os.path.isfile(weights):
            raise WeightsError(f"weights file {weights!r} not found; pass 'pretrained', "
                               "'random', or a readable .pth path")
        model = wide_resnet50_2(weights=None)
        model.load_state_dict(torch.load(weights, map_location="cpu"))
    trunk = torch.nn.Sequential(model.conv1, model.bn1, model.relu, model.maxpool,
                                model.layer1, model.layer2).eval()
    return trunk.to(device if device is not None else torch.device("cuda"))


def normalize(images: torch.Tensor) -> torch.Tensor:
    """(B, 3, H, W) uint8 [0, 255] or float [0, 1] -> ImageNet-normalised float32
    (export.py:104-113 after the resize)."""
    x = images.float() / 255.0 if images.dtype == torch.uint8 else images.float()
    mean = torch.tensor(MEAN, device=x.device)[:, None, None]
    std = torch.tensor(STD, device=x.device)[:, None, None]
    return (x - mean) / std


@torch.no_grad()
def extract_features(trunk: torch.nn.Module, images: torch.Tensor,
                     resolution: int | None = None, chunk: int = 16) -> torch.Tensor:
    """Images (B, 3, H, W) on the GPU -> (B, 512, R/8, R/8) float32 features.

    ``resolution``: bilinear resize to R x R first (the reference resizes with
    PIL before the trunk; torch's bilinear with antialias differs from PIL's
    in the last bits, so pass pre-resized images for exact parity).
    """
    x = images
    if resolution is not None and tuple(x.shape[-2:]) != (resolution, resolution):
        x = torch.nn.functional.interpolate(x.float(), size=(resolution, resolution),
                                            mode="bilinear", antialias=True,
                                            align_corners=False)
    prev = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = False  # fp32 features, as the reference's
    try:
        out = [trunk(normalize(x[i:i + chunk])).float() for i in range(0, x.shape[0], chunk)]
    finally:
        torch.backends.cudnn.allow_tf32 = prev
    return torch.cat(out).contiguous()
