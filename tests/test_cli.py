"""The CLI (reference cli.py) on the GPU path: parser, --config, exit codes
(CPU), and detect / evaluate over a small MVTec-layout tree of QTF1 feature
files against the oracle (GPU)."""

from __future__ import annotations

import io
import json
import os
from contextlib import redirect_stderr, redirect_stdout

import numpy as np
import pytest

from paper_2510_15602_b200 import cli
from paper_2510_15602_b200.tensor_io import (DatasetIndexError, load_dataset, load_mask,
                                             write_tensor)


def run(argv):
    out, err = io.StringIO(), io.StringIO()
    with redirect_stdout(out), redirect_stderr(err):
        rc = cli.main(argv)
    return rc, out.getvalue(), err.getvalue()


def test_cli_usage_errors_exit_2(tmp_path):
    assert run([])[0] == 2
    assert run(["detect"])[0] == 2  # --image / --features required
    assert run(["detect", "--image", "x.png"])[0] == 2  # filter-bank front end: not here
    assert run(["synth", "--out", str(tmp_path)])[0] == 2
    assert run(["evaluate", "--dataset", str(tmp_path), "--classes", "a"])[0] == 2
    assert run(["detect", "--features", "f.qtf", "--config"])[0] == 2
    bad = tmp_path / "bad.cfg"
    bad.write_text("no equals sign\n")
    assert run(["--config", str(bad), "detect", "--features", "f.qtf"])[0] == 2
    assert run(["--version"])[0] == 0


def test_cli_config_file_sets_defaults(tmp_path):
    cfgf = tmp_path / "run.cfg"
    cfgf.write_text("# comment\npatch-size = 5\nbins=8\nreference = quan-mean\n")
    p = cli.build_parser()
    for sp in p._subparsers._group_actions[0].choices.values():
        known = {a.dest for a in sp._actions}
        sp.set_defaults(**{k: v for k, v in cli._load_config_file(str(cfgf)).items()
                           if k in known})
    a = p.parse_args(["detect", "--features", "f.qtf", "--bins", "4"])
    assert (a.patch_size, a.bins, a.reference) == (5, 4, "quan-mean")
    c = cli._pipeline_config(a)
    assert (c.patch_size, c.n_bins, c.reference_mode) == (5, 4, "quan-mean")


def _png(path, arr):
    from PIL import Image
    os.makedirs(os.path.dirname(path), exist_ok=True)
    Image.fromarray(arr).save(path)


def make_tree(root, rng, c=16, h=16, w=16, scale=4):
    """root/tex/test/{good,cut}/NNN.png, ground_truth/cut/NNN_mask.png and
    features/tex/<defect>/NNN.qtf (+ scale sidecar)."""
    feats = {}
    for defect, n in (("cut", 3), ("good", 2)):
        for i in range(n):
            stem = f"{i:03d}"
            _png(os.path.join(root, "tex", "test", defect, stem + ".png"),
                 np.zeros((h * scale, w * scale), np.uint8))
            x = np.maximum(rng.standard_normal((c, h, w)), 0).astype(np.float32)
            m = np.zeros((h * scale, w * scale), np.uint8)
            if defect != "good":
                y0, x0 = rng.integers(8, h * scale - 24, 2)
                m[y0:y0 + 14, x0:x0 + 18] = 255
                x[:, y0 // scale:(y0 + 14) // scale, x0 // scale:(x0 + 18) // scale] += 1.5
                _png(os.path.join(root, "tex", "ground_truth", defect, stem + "_mask.png"), m)
            fp = os.path.join(root, "features", "tex", defect, stem + ".qtf")
            os.makedirs(os.path.dirname(fp), exist_ok=True)
            write_tensor(x, fp)
            with open(fp + ".json", "w") as fh:
                json.dump({"scale": scale}, fh)
            feats[(defect, stem)] = (x, m > 0)
    return feats


def test_dataset_index_and_masks(tmp_path):
    make_tree(str(tmp_path), np.random.default_rng(0))
    idx = load_dataset(str(tmp_path), "tex")
    assert [(s.defect_type, os.path.basename(s.image_path), s.is_anomalous) for s in idx] == [
        ("cut", "000.png", True), ("cut", "001.png", True), ("cut", "002.png", True),
        ("good", "000.png", False), ("good", "001.png", False)]
    assert idx[3].mask_path is None
    m = load_mask(idx[0].mask_path)
    assert m.dtype == bool and m.shape == (64, 64) and m.any()
    m2 = load_mask(idx[0].mask_path, size=(32, 32))
    np.testing.assert_array_equal(m2, m[::2, ::2])  # half-pixel centres 2i + .5, round-half-even
    os.remove(idx[1].mask_path)
    with pytest.raises(DatasetIndexError):
        load_dataset(str(tmp_path), "tex")


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["upsample-scores", "downsample-mask"])
def test_cli_evaluate_matches_oracle(tmp_path, mode):
    from oracle import qfca_oracle as O
    feats = make_tree(str(tmp_path), np.random.default_rng(1))
    rc, out, err = run(["evaluate", "--dataset", str(tmp_path), "--classes", "tex",
                        "--features-dir", str(tmp_path / "features"), "--patch-size", "5",
                        "--mask-mode", mode])
    assert rc == 0, err
    got = json.loads(out)["tex"]
    samples = []
    for (defect, _), (x, m) in sorted(feats.items()):
        sc, _, _ = O.detect(x, patch_size=5)
        if mode == "upsample-scores":
            samples.append((O.upsample_scores(sc, 64, 64), m, defect != "good", 2 * 4))
        else:
            samples.append((sc, cli._majority_downsample(m, 4), defect != "good", 2))
    s_, l_ = O.metrics_pooled(samples)
    want = {"pro": O.pro_at_fpr(samples), "auroc_s": O.rank_auroc(s_, l_),
            "f1": O.f1_optimal(s_, l_), "auroc_c": O.auroc_image(samples)}
    for k, v in want.items():
        assert got[k] == pytest.approx(v, abs=2e-3), k
    assert got["n_images"] == 5


@pytest.mark.gpu
def test_cli_detect_features(tmp_path):
    from oracle import qfca_oracle as O
    from paper_2510_15602_b200.tensor_io import read_tensor
    rng = np.random.default_rng(2)
    x = np.maximum(rng.standard_normal((24, 20, 22)), 0).astype(np.float32)
    fp = str(tmp_path / "f.qtf")
    write_tensor(x, fp)
    rc, out, err = run(["detect", "--features", fp, "--out", str(tmp_path / "h.qtf"),
                        "--full-resolution", "--manifest", str(tmp_path / "m.json")])
    assert rc == 0, err
    sc, img, _ = O.detect(x)
    assert json.loads(out)["image_score"] == pytest.approx(img, rel=1e-4)
    heat = read_tensor(str(tmp_path / "h.qtf"))
    assert heat.shape == (160, 176) and heat.dtype == np.float32  # default scale 8
    np.testing.assert_allclose(heat, O.upsample_scores(sc, 160, 176).astype(np.float32),
                               atol=1e-4 * np.abs(sc).max())
    man = json.load(open(tmp_path / "m.json"))
    assert man["inputs"] == [fp] and man["config"]["n_bins"] == 16
    rc, _, _ = run(["detect", "--features", fp, "--out", str(tmp_path / "h.pgm")])
    assert rc == 0 and open(tmp_path / "h.pgm", "rb").read(2) == b"P5"
    rc, out, _ = run(["bench", "--suite", "patch", "--sizes", "32", "--kernels", "3,9",
                      "--repeats", "2"])
    assert rc == 0 and out.splitlines()[0] == "suite,param,median_ms,p10,p90"
    assert len(out.splitlines()) == 3
