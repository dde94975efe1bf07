"""QTF1 feature files: byte layout and validation against files written by the
reference's own writer (tests/golden/make_qtf1.py), CPU only."""
import os

import numpy as np
import pytest

from paper_2510_15602_b200 import tensor_io as T

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_reads_reference_files():
    ref = {"feats": np.load(os.path.join(G, "qtf1_feats.npy")),
           "img": np.load(os.path.join(G, "qtf1_img.npy"))}
    a = T.read_tensor(os.path.join(G, "qtf1_features_6x5x7.qtf"))
    assert a.dtype == np.float32 and a.shape == (6, 5, 7)
    np.testing.assert_array_equal(a, ref["feats"])
    b = T.read_tensor(os.path.join(G, "qtf1_uint8_3x4x2.qtf"))
    assert b.dtype == np.uint8
    np.testing.assert_array_equal(b, ref["img"])


def test_writes_reference_bytes(tmp_path):
    ref = {"feats": np.load(os.path.join(G, "qtf1_feats.npy")),
           "img": np.load(os.path.join(G, "qtf1_img.npy"))}
    for name, arr in (("qtf1_features_6x5x7.qtf", ref["feats"]), ("qtf1_uint8_3x4x2.qtf", ref["img"])):
        p = tmp_path / name
        T.write_tensor(arr, p)
        assert p.read_bytes() == open(os.path.join(G, name), "rb").read()


def test_validation_errors(tmp_path):
    good = open(os.path.join(G, "qtf1_features_6x5x7.qtf"), "rb").read()
    cases = [(b"QTF2" + good[4:], T.BadMagicError), (good[:5], T.TruncatedError),
             (good[:10], T.TruncatedError), (good[:-4], T.TruncatedError),
             (good + b"\0", T.TensorFormatError),
             (good[:4] + bytes([9]) + good[5:], T.UnsupportedDtypeError),
             (good[:5] + bytes([5]) + good[6:], T.TensorFormatError)]
    for i, (raw, err) in enumerate(cases):
        p = tmp_path / f"bad{i}.qtf"
        p.write_bytes(raw)
        with pytest.raises(err):
            T.read_tensor(p)
    with pytest.raises(T.UnsupportedDtypeError):
        T.write_tensor(np.zeros((2, 2), np.float64), tmp_path / "f64.qtf")
