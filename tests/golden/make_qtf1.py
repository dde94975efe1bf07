"""QTF1 fixtures written by THE REFERENCE's own writer (qfca.tensor_io.write_tensor,
tensor_io.py:79-93); build container only:  python tests/golden/make_qtf1.py"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from qfca import tensor_io as T  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(2510)
feats = np.maximum(rng.standard_normal((6, 5, 7)), 0).astype(np.float32)
T.write_tensor(T.Tensor.from_array(feats), os.path.join(OUT, "qtf1_features_6x5x7.qtf"))
img = rng.integers(0, 256, (3, 4, 2), dtype=np.uint8)
T.write_tensor(T.Tensor.from_array(img), os.path.join(OUT, "qtf1_uint8_3x4x2.qtf"))
np.save(os.path.join(OUT, "qtf1_feats.npy"), feats)
np.save(os.path.join(OUT, "qtf1_img.npy"), img)
print("wrote QTF1 fixtures")
