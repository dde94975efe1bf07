"""B200-native QFCA scoring path (arXiv 2510.15602), drop-in for ``qfca``.

The public names follow the reference package's API (reference
pkg/src/qfca/__init__.py:12-28, hot-path subset): feature preprocessing
(FeatureMap, PcaModel, pca_fit, pca_residual), the quantizer
(fit_quantizer, bin_indices, patch_histograms, select_reference) and the
scorer (PipelineConfig, AnomalyMap, detect, ...).  Every computation runs in
hand-written sm_100a CUDA kernels (libqfca_b200.so, C-ABI in
include/qfca_b200.h); there is no CPU fallback.  ``detect_batch`` is the
batched device entry point.
"""

__version__ = "0.1.0"

from .features import (FeatureMap, FormatError, PcaModel, gaussian_blur, pca_fit,
                       pca_residual)
from .pooling import (SummedAreaTable, box_average, box_average_stack, box_sum, build_sat,
                      naive_box_average, pad_plane)
from .quantize import (REFERENCE_MODES, BinIndexMap, HistogramField, Quantizer,
                       ReferenceHistogram, bin_indices, fit_quantizer, patch_histograms,
                       select_reference)
from .scoring import (AnomalyMap, DetectResult, PipelineConfig, aggregate_channels,
                      associate_errors, bin_error_maps, channel_error_maps, detect,
                      detect_batch, fused_supported, image_score_of, smooth_scores,
                      upsample_batch, upsample_scores)
from .transport import (IllConditionedError, MassError, mismatch_batch,
                        quantized_mismatch)
from .pipeline import DetectPipeline, HostResult
from . import exporter, tensor_io  # feature backbone on the GPU, QTF1 feature files
from . import metrics  # PRO / AUROC / F1 / components on the GPU (metrics.py)
from .metrics import EvalSample, MetricReport

__all__ = [
    "FeatureMap", "FormatError", "PcaModel", "gaussian_blur", "pca_fit", "pca_residual",
    "box_average", "box_average_stack", "SummedAreaTable", "box_sum", "build_sat",
    "naive_box_average", "pad_plane", "REFERENCE_MODES", "BinIndexMap", "HistogramField",
    "Quantizer", "ReferenceHistogram", "bin_indices", "fit_quantizer", "patch_histograms",
    "select_reference", "AnomalyMap", "DetectResult", "PipelineConfig", "aggregate_channels",
    "associate_errors", "bin_error_maps", "channel_error_maps", "detect", "detect_batch",
    "fused_supported", "image_score_of", "smooth_scores", "upsample_batch",
    "upsample_scores", "IllConditionedError", "MassError", "mismatch_batch",
    "quantized_mismatch", "DetectPipeline", "HostResult", "exporter", "tensor_io",
    "metrics", "EvalSample", "MetricReport",
]
