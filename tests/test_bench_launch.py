"""CPU tests of bench.py's multi-rank entry and the reference arm's machinery.

`bench.py --gpus 2 --dry-run` must re-launch itself under torch.distributed.run
(two gloo ranks on this host), split the global batch across them and print ONE
JSON line from rank 0 with n_gpus = 2.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_bench_self_launches_two_ranks():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--dry-run", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1, p.stdout
    line = lines[0]
    assert line["n_gpus"] == 2
    assert line["images_all_ranks_per_step"] == line["config"]["global_batch"] == 512
    assert line["config"]["images_per_gpu"] == 256
    assert line["scaling"] == "strong" and line["warmup"] >= 3


def test_bench_default_is_configs2():
    sys.path.insert(0, ROOT)
    import bench
    size, images, is_global, pca_k, scaling, _ = bench.WORKLOADS[bench.DEFAULT_WORKLOAD]
    assert (size, images, is_global, pca_k, scaling) == (1024, 512, True, 0, "strong")


def test_reference_pool_runs_the_installed_reference():
    sys.path.insert(0, ROOT)
    from baseline import refpool
    why = refpool.available()
    if why is not None:
        pytest.skip(why)
    x = np.maximum(np.random.default_rng(0).standard_normal((2, 6, 16, 16)), 0)
    x = x.astype(np.float32)
    pool = refpool.ReferencePool(x, 0, 128, workers=2)
    try:
        wall, per = pool.step()
    finally:
        pool.close()
    assert len(per) == 2 and wall > 0
    # the workers ran the reference from baseline/_ref, whose detect the oracle pins
    from oracle import qfca_oracle as O
    qfca = refpool._import_qfca()
    a = qfca.detect(qfca.FeatureMap(x[0], 8), qfca.PipelineConfig())
    ref, img, _ = O.detect(x[0])
    assert np.abs(a.scores - ref).max() <= 1e-4 * np.abs(ref).max()
