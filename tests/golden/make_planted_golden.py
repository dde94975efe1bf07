"""PRO / AUROC / F1 goldens on planted-defect textures, made by RUNNING THE
REFERENCE ITSELF end to end (build container only):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_planted_golden.py

For each kind (noise / tiles / stripes) the reference's synthetic generator
(synth.py:42-115, the rng sequence of generate_class, synth.py:127-144) makes
10 textures of 128 x 128 (the first 3 clean, 7 with a planted square); the
image goes through a uint8 round trip as in _save_png / load_image
(synth.py:117-124, tensor_io.py:161-183), features come from the reference's
own filter bank (features.py:103-129, 39 channels at stride 4 -- the CLI's
`qfca evaluate --image` path), then detect (scoring.py:235-299) with the
default config, upsample_scores to 128 x 128, and the reference metrics
(metrics.py:149-206) exactly as evaluate_class forms its samples
(cli.py:141-170, border = cfg.border * scale).

Writes tests/golden/planted_filterbank.npz (features, masks, labels, feature
maps, upsampled maps as float32 -- lossless: upsample_scores rounds through
float32 -- and the per-class metric rows).
"""

from __future__ import annotations

import os
import sys
import zlib

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF_SRC)

from qfca import metrics, scoring, synth  # noqa: E402
from qfca.features import extract_filterbank  # noqa: E402

KINDS = ("noise", "tiles", "stripes")
SIZE, N_IMAGES, N_GOOD, SEED = 128, 10, 3, 0


def main():
    cfg = scoring.PipelineConfig()
    out = {"kinds": np.array(KINDS), "size": np.int64(SIZE)}
    for kind in KINDS:
        rng = np.random.default_rng([SEED, zlib.crc32(kind.encode())])
        feats, masks, labels, fmaps, ups, img_scores = [], [], [], [], [], []
        samples = []
        for i in range(N_IMAGES):
            image = synth._texture(kind, rng, SIZE)
            mask = np.zeros((SIZE, SIZE), dtype=bool)
            if i >= N_GOOD:
                mask = synth._anomaly_mask("square", rng, SIZE, 0.02)
                image = synth._plant_anomaly(image, mask, kind, rng)
            u8 = np.round(np.asarray(image).transpose(1, 2, 0) * 255).astype(np.uint8)
            image = u8.transpose(2, 0, 1).astype(np.float64) / 255.0
            f = extract_filterbank(image)
            amap = scoring.detect(f, cfg)
            up = scoring.upsample_scores(amap.scores, SIZE, SIZE)
            assert np.array_equal(up, up.astype(np.float32).astype(np.float64))
            feats.append(f.values)
            masks.append(mask)
            labels.append(i >= N_GOOD)
            fmaps.append(amap.scores)
            ups.append(up.astype(np.float32))
            img_scores.append(amap.image_score)
            samples.append(metrics.EvalSample(scores=up, mask=mask, image_label=i >= N_GOOD,
                                              border=cfg.border * f.scale))
        row = metrics.MetricReport().add_class(kind, samples)
        out[f"{kind}/features"] = np.stack(feats)
        out[f"{kind}/masks"] = np.stack(masks)
        out[f"{kind}/labels"] = np.array(labels)
        out[f"{kind}/maps"] = np.stack(fmaps)
        out[f"{kind}/upsampled"] = np.stack(ups)
        out[f"{kind}/image_scores"] = np.array(img_scores)
        for k in ("pro", "auroc_s", "f1", "auroc_c"):
            out[f"{kind}/{k}"] = np.float64(row[k])
        out[f"{kind}/border"] = np.int64(cfg.border * f.scale)
        out[f"{kind}/scale"] = np.int64(f.scale)
        print(kind, {k: round(row[k], 6) for k in ("pro", "auroc_s", "f1", "auroc_c")})
    path = os.path.join(OUT, "planted_filterbank.npz")
    np.savez_compressed(path, **out)
    print(path)


if __name__ == "__main__":
    main()
