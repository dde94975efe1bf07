"""Golden vectors for the pooling API, made by RUNNING THE REFERENCE ITSELF
(qfca.pooling, /root/reference/pkg/src/qfca/pooling.py).  Build container only:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_pooling_golden.py

Writes tests/golden/pooling.npz: inputs and the reference's outputs of
pad_plane, build_sat, box_sum, box_average, box_average_stack and
naive_box_average over every pad mode, several kernels, tiny / degenerate
planes (1 x w, h x 1, 1 x 1), margins larger than the plane, and float32 /
float64 / integer inputs.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF_SRC)

from qfca import pooling  # noqa: E402


def main():
    rng = np.random.default_rng(20261019)
    planes = {
        "f32_9x11": rng.standard_normal((9, 11)).astype(np.float32),
        "f64_16x13": rng.random((16, 13)) * 1e3 - 300.0,
        "i32_7x5": rng.integers(-50, 50, (7, 5)).astype(np.int32),
        "u8_6x8": rng.integers(0, 255, (6, 8)).astype(np.uint8),
        "f32_1x7": rng.standard_normal((1, 7)).astype(np.float32),
        "f32_6x1": rng.standard_normal((6, 1)).astype(np.float32),
        "f64_1x1": np.array([[2.5]]),
        "f64_2x2": np.array([[1.0, 2.0], [3.0, 4.0]]),
        "f32_3x4": rng.standard_normal((3, 4)).astype(np.float32),
    }
    out = {}
    for name, p in planes.items():
        out[f"in/{name}"] = p
        for pad in ("zero", "reflect", "wrap"):
            for margin in (0, 1, 3, 9):
                out[f"pad/{name}/{pad}/{margin}"] = pooling.pad_plane(p, margin, pad)
                sat = pooling.build_sat(p, margin=margin, pad=pad)
                out[f"sat/{name}/{pad}/{margin}"] = sat.cumsum
                for k in (1, 3, 5):
                    r = k // 2
                    if pad != "zero" and margin < r:
                        continue
                    vals = [pooling.box_sum(sat, cx, cy, k, pad=pad)
                            for cx in range(p.shape[0]) for cy in range(p.shape[1])]
                    out[f"boxsum/{name}/{pad}/{margin}/{k}"] = np.asarray(vals)
            for k in (1, 3, 5, 9, 31):
                out[f"avg/{name}/{pad}/{k}"] = pooling.box_average(p, k, pad)
                out[f"naive/{name}/{pad}/{k}"] = pooling.naive_box_average(p, k, pad)
    stacks = {
        "f64_3x10x12": rng.standard_normal((3, 10, 12)),
        "f32_2x1x9": rng.standard_normal((2, 1, 9)).astype(np.float32),
        "f32_2x7x1": rng.standard_normal((2, 7, 1)).astype(np.float32),
        "f64_4x5x5": rng.random((4, 5, 5)),
    }
    for name, s in stacks.items():
        out[f"in/{name}"] = s
        for pad in ("zero", "reflect", "wrap"):
            for k in (1, 3, 7, 11):
                out[f"stack/{name}/{pad}/{k}"] = pooling.box_average_stack(s, k, pad)
    path = os.path.join(OUT, "pooling.npz")
    np.savez_compressed(path, **out)
    print(path, len(out))


if __name__ == "__main__":
    main()
