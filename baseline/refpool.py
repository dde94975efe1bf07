"""Times the UNMODIFIED reference (`qfca`, installed into baseline/_ref from
/root/reference/pkg) on the host's cores: the reference arm of bench.py and
the `cpu_baseline` leg of the GPU arm.

Timed call per image, as the reference's own callers do it
(cli.py:97-131 `cmd_detect` with --full-resolution):
    amap = qfca.detect(qfca.FeatureMap(values, scale=8), cfg)   # scoring.py:235-299
    qfca.upsample_scores(amap.scores, S, S)                      # scoring.py:149-152

Two modes:
  * "pool"        -- mode (ii): os.cpu_count() worker processes, each with
                     NUMBA/OMP/OPENBLAS/MKL_NUM_THREADS=1, one image per worker
                     per step (images are independent);
  * "as_shipped"  -- mode (i): one process, the reference's defaults (its hot
                     loop is single-threaded Numba; BLAS threads for the PCA).
Numba JIT compilation is warmed (and cached under NUMBA_CACHE_DIR) before any
timed region.  Inputs are shared with the workers through a .npy file in /tmp
(memory-mapped, read from the page cache).  Nothing here touches the GPU.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
CACHE_DIR = os.path.join(tempfile.gettempdir(), "qfca_ref_numba_cache")

_W = {}


def available() -> str | None:
    """None when the installed reference imports, else the reason."""
    if not os.path.isdir(os.path.join(REF_DIR, "qfca")):
        return f"reference not installed in {REF_DIR}"
    try:
        import numba  # noqa: F401
    except Exception as e:  # pragma: no cover - depends on the box
        return f"numba missing: {e}"
    return None


def _import_qfca():
    os.environ.setdefault("NUMBA_CACHE_DIR", CACHE_DIR)
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import qfca
    if not os.path.abspath(qfca.__file__).startswith(REF_DIR):
        raise RuntimeError(f"qfca imported from {qfca.__file__}, not {REF_DIR}")
    return qfca


def _warm(qfca, pca_k: int):
    import numpy as np
    rng = np.random.default_rng(0)
    v = np.maximum(rng.standard_normal((max(pca_k + 2, 4), 12, 12)), 0).astype(np.float32)
    cfg = qfca.PipelineConfig(pca_components=pca_k)
    a = qfca.detect(qfca.FeatureMap(v, 8), cfg)
    qfca.upsample_scores(a.scores, 96, 96)


def _init_worker(path: str, pca_k: int, size: int):
    qfca = _import_qfca()
    import numpy as np
    _W["qfca"] = qfca
    _W["x"] = np.load(path, mmap_mode="r")
    _W["cfg"] = qfca.PipelineConfig(pca_components=pca_k)
    _W["size"] = size
    _warm(qfca, pca_k)


def _one(i: int):
    import numpy as np
    qfca, x = _W["qfca"], _W["x"]
    v = np.array(x[i % x.shape[0]])  # page cache -> private copy (outside the timer)
    t0 = time.perf_counter()
    amap = qfca.detect(qfca.FeatureMap(v, 8), _W["cfg"])
    qfca.upsample_scores(amap.scores, _W["size"], _W["size"])
    return time.perf_counter() - t0, float(amap.image_score)


def _ready(_):
    return os.getpid()


def _single_thread_env():
    env = {k: "1" for k in ("NUMBA_NUM_THREADS", "OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS",
                            "MKL_NUM_THREADS")}
    env["NUMBA_CACHE_DIR"] = CACHE_DIR
    return env


class ReferencePool:
    """os.cpu_count() spawned workers running the reference, one image each per step."""

    def __init__(self, x, pca_k: int, size: int, workers: int | None = None):
        import numpy as np
        self.workers = workers or os.cpu_count() or 1
        # compile once in this process so the workers load the Numba cache
        _warm(_import_qfca(), pca_k)
        fd, self.path = tempfile.mkstemp(suffix=".npy", prefix="qfca_ref_in_")
        os.close(fd)
        np.save(self.path, np.ascontiguousarray(x, dtype=np.float32))
        self.n_inputs = int(x.shape[0])
        saved = {k: os.environ.get(k) for k in _single_thread_env()}
        os.environ.update(_single_thread_env())  # inherited by the spawned workers
        try:
            ctx = mp.get_context("spawn")
            self.pool = ctx.Pool(self.workers, initializer=_init_worker,
                                 initargs=(self.path, pca_k, size))
            self.pool.map(_ready, range(self.workers), chunksize=1)  # all initialised
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        self._next = 0

    def step(self, images: int | None = None):
        """Score `images` (default: one per worker) -> (wall seconds, per-image seconds)."""
        n = images or self.workers
        idx = list(range(self._next, self._next + n))
        self._next += n
        t0 = time.perf_counter()
        res = self.pool.map(_one, idx, chunksize=1)
        return time.perf_counter() - t0, [r[0] for r in res]

    def close(self):
        self.pool.terminate()
        self.pool.join()
        try:
            os.unlink(self.path)
        except OSError:
            pass


def as_shipped_seconds(v, pca_k: int, size: int) -> float:
    """Mode (i): one image through the reference in this process, its defaults."""
    qfca = _import_qfca()
    _warm(qfca, pca_k)
    cfg = qfca.PipelineConfig(pca_components=pca_k)
    t0 = time.perf_counter()
    amap = qfca.detect(qfca.FeatureMap(v, 8), cfg)
    qfca.upsample_scores(amap.scores, size, size)
    return time.perf_counter() - t0


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
