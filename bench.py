"""QFCA scoring throughput on B200 (driver contract: one JSON line on rank 0).

Default workload = BASELINE.json configs[2], the configuration the north-star
1/2/4/8-GPU curve is quoted on: QFCA on a batch of 512 synthetic 1024x1024
textures (WRN50-2 random-init block-2 features, 512 x 128 x 128 fp32 per
image), default bins / patch size, the 512 images split over the N ranks with
no communication (strong scaling: 512/N per rank).  A step = one pass of the
path over the rank's images: min/max -> bins -> sort-free reference -> fused
histogram / transport / association / channel sum -> channel mean, smoothing,
image scores -> bilinear upsampling to image resolution.

Other workloads: `--workload qfca_plus512` (configs[1]: QFCA + PCA k=10,
64 x 512^2 per GPU) and `--workload qfca8192` (configs[4]: one 8192^2 texture,
channels sharded over the ranks, one all-reduce of the channel-sum map).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

`--gpus N` without a torchrun environment re-launches itself under
`torch.distributed.run` with N ranks (one process per GPU).  `--dry-run`
replaces the GPU step with a host stand-in on the gloo backend (used by the CPU
test of the multi-rank entry).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# name: (image size, images, images-are-global, pca components, scaling, label)
WORKLOADS = {
    "qfca1024": (1024, 512, True, 0, "strong",
                 "configs[2]: QFCA, batch 512 of 1024x1024 synthetic textures (WRN50-2 "
                 "random-init block-2 features) split over the GPUs, no comms"),
    "qfca_plus512": (512, 64, False, 10, "weak",
                     "configs[1]: QFCA + PCA (k=10), batch 64 of 512x512 synthetic textures "
                     "per GPU, WRN50-2 random-init block-2 features"),
    "qfca8192": (8192, 1, True, 0, "strong",
                 "configs[4]: one 8192x8192 synthetic texture (512 x 1024^2 WRN50-2 "
                 "random-init block-2 features), channels sharded across the ranks, one "
                 "all-reduce of the channel-sum map"),
}
DEFAULT_WORKLOAD = "qfca1024"
METRIC = "images/sec (megapixels/sec) of QFCA scoring at 1/2/4/8 B200; % of HBM roofline"
CHUNK = 64  # images per detect_batch call inside a step


def alg_bytes_per_image(size: int, pca: bool, channels: int = 512, stride: int = 8) -> int:
    """features read once + feature-res map + full-res map
    (+ one more feature read for the PCA covariance pass)."""
    h = w = size // stride
    b = 4 * channels * h * w + 4 * h * w + 4 * size * size
    return b + (4 * channels * h * w if pca else 0)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, enabled: bool = True):
        self.index = index
        self.enabled = enabled
        self.samples = []
        self._proc = None
        self._thr = None
        self._live = False

    def _run(self):
        for line in self._proc.stdout:
            if self._live and line.strip():
                self.samples.append([p.strip() for p in line.split(",")])

    def __enter__(self):
        # one long-running nvidia-smi sampling every 200 ms (50 ms polling was
        # measured to perturb the timed GPU work)
        if self.enabled:
            try:
                self._proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits", "-lms",
                     os.environ.get("QFCA_BENCH_SMI_MS", "200")],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self._live = True  # samples from just before the region count too
                self._thr = threading.Thread(target=self._run, daemon=True)
                self._thr.start()
                time.sleep(0.3)  # let the first sample land before the timed region
            except Exception:
                self._proc = None
        self._live = True
        return self

    def __exit__(self, *a):
        self._live = False
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
            self._thr.join(timeout=5)

    def summary(self):
        import statistics
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ------------------------------------------------------------------ launch
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(n: int) -> int:
    """Re-run this command under torch.distributed.run with n ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def init_dist(ws: int, local: int, backend: str):
    import torch
    import torch.distributed as dist
    if ws == 1:
        return None
    if backend == "nccl":
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("gloo")
    return dist


def max_over_ranks(x: float, dist, dev) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ CPU baselines
def reference_cpu_baseline(x_host, pca_k: int, size: int, budget_s: float = 25.0):
    """The unmodified reference (baseline/_ref) on all host cores (mode ii), one
    image per worker per round, bounded to ~budget_s; mode (i) beside it."""
    from baseline import refpool
    why = refpool.available()
    if why is not None:
        return None, why
    pool = refpool.ReferencePool(x_host, pca_k, size)
    try:
        done, wall, rounds, per = 0, 0.0, 0, []
        while True:
            el, times = pool.step()
            done += len(times)
            wall += el
            per += times
            rounds += 1
            if wall >= budget_s or rounds >= 4 or wall / rounds * (rounds + 1) > 2 * budget_s:
                break
    finally:
        pool.close()
    single = refpool.as_shipped_seconds(x_host[0], pca_k, size)
    return {"value": done / wall, "unit": "images/s", "cores": pool.workers,
            "kind": "reference",
            "sample": f"{done} images ({size}x{size}, 512 ch) in {rounds} rounds of one "
                      f"image per worker; qfca.detect + upsample_scores from baseline/_ref, "
                      f"{pool.workers} processes x 1 thread (mode ii)",
            "cpu_model": refpool.cpu_model(),
            "per_image_s_median": sorted(per)[len(per) // 2],
            "as_shipped": {"value": 1.0 / single, "unit": "images/s", "cores": 1,
                           "sample": "1 image, one process, reference defaults (mode i)"}}, None


def port_cpu_baseline(x_host, pca_k: int, size: int, max_seconds: float = 10.0):
    """The C/NumPy oracle restatement (kind "port"), OpenMP over channels."""
    import numpy as np
    from oracle import qfca_oracle as O
    O.set_threads(os.cpu_count() or 1)
    done, t0 = 0, time.perf_counter()
    while True:
        O.detect(np.ascontiguousarray(x_host[done % x_host.shape[0]]), pca_components=pca_k)
        O.upsample_scores(np.zeros((size // 8, size // 8)), size, size)
        done += 1
        el = time.perf_counter() - t0
        if el >= max_seconds or done >= x_host.shape[0]:
            break
    return {"value": done / el, "unit": "images/s", "cores": O.num_threads(), "kind": "port",
            "sample": f"{done} images ({size}x{size}, 512 ch), C oracle (OpenMP over "
                      f"channels) + NumPy PCA"}


# ------------------------------------------------------------------ reference arm
def run_reference_arm(args, ws, rank, config, size, pca_k, mp_per_image):
    """--impl reference: the unmodified reference on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import numpy as np
    import torch
    from baseline import refpool
    import workloads
    cores = os.cpu_count() or 1
    dev = "cuda" if torch.cuda.is_available() and not args.dry_run else "cpu"
    n_in = min(cores, 16)
    if args.workload == "qfca8192":
        # one 8192^2 image: its 512 channels are independent up to the channel mean,
        # so a step scores one 1024^2 channel per worker; img/s extrapolates x512/cores
        feats, _ = workloads.make_features(1, size, seed=1000, device=dev)
        x_host = feats[0, :n_in].cpu().numpy()[:, None]
        per_image_units = feats.shape[1]
    else:
        feats, _ = workloads.make_features(n_in, size, seed=1000, device=dev)
        x_host = feats.cpu().numpy()
        per_image_units = 1
    del feats
    why = refpool.available()
    line = {"metric": METRIC, "impl": "reference", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": config["scaling"],
            "vs_baseline": None, "dtype": "f32 in / f64 (reference NumPy/Numba)",
            "data": "synthetic", "config": config}
    up_size = size if per_image_units == 1 else x_host.shape[-1]  # per-channel units
    if why is not None:  # the oracle port stands in, and says so
        if per_image_units == 1:
            cpu = port_cpu_baseline(x_host, pca_k, size, max_seconds=20.0)
        else:
            cpu = port_cpu_baseline(x_host[:, 0][None], 0, up_size, max_seconds=20.0)
            cpu["value"] *= x_host.shape[0] / per_image_units  # one image = all channels
        cpu["why_not_reference"] = why
        line.update({"value": cpu["value"], "unit": "images/s", "cpu_baseline": cpu,
                     "e2e": {"value": cpu["value"], "unit": "images/s",
                             "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
        print(json.dumps(line), flush=True)
        return
    pool = refpool.ReferencePool(x_host, pca_k, up_size)
    try:
        for _ in range(args.warmup):
            pool.step()
        total_s, imgs = 0.0, 0
        per = []
        for _ in range(args.steps):
            el, times = pool.step()
            total_s += el
            imgs += len(times)
            per += times
    finally:
        pool.close()
    units_per_s = imgs / total_s
    ips = units_per_s / per_image_units
    sample = (f"each step: one {size}x{size} image (512 ch) per worker, {pool.workers} "
              f"workers" if per_image_units == 1 else
              f"each step: one 1024x1024 channel of the 8192^2 image per worker, "
              f"{pool.workers} workers; img/s = channels/s / {per_image_units}")
    line.update({"value": ips, "unit": "images/s", "mp_per_s": ips * mp_per_image,
                 "ms_per_step": 1e3 * total_s / max(args.steps, 1),
                 "cpu_baseline": {"value": ips, "unit": "images/s", "cores": pool.workers,
                                  "kind": "reference", "sample": sample,
                                  "cpu_model": refpool.cpu_model(),
                                  "per_image_s_median": sorted(per)[len(per) // 2]},
                 "e2e": {"value": ips, "unit": "images/s", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0}})
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ dry run (CPU, gloo)
def run_dry(args, ws, rank, config, per_rank):
    """Host stand-in for the GPU step: exercises the launch, the image split, the
    barrier and the max-over-ranks timing on the gloo backend."""
    import numpy as np
    import torch
    dist = init_dist(ws, 0, "gloo")
    x = np.random.default_rng(rank).standard_normal((per_rank, 4, 8, 8)).astype(np.float32)

    def step():
        return float(np.maximum(x, 0).sum())

    for _ in range(max(3, args.warmup)):
        step()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = max_over_ranks(time.perf_counter() - t0, dist, "cpu")
    cnt = torch.tensor([per_rank], dtype=torch.int64)
    if dist is not None:
        dist.all_reduce(cnt)
    if rank == 0:
        total = int(cnt[0]) * args.steps
        print(json.dumps({"metric": METRIC, "value": total / el, "unit": "images/s",
                          "n_gpus": ws, "steps": args.steps, "warmup": max(3, args.warmup),
                          "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
                          "scaling": config["scaling"], "vs_baseline": None, "dtype": "f32",
                          "data": "synthetic (dry run: host stand-in, no GPU work)",
                          "config": config, "images_all_ranks_per_step": int(cnt[0]),
                          "dry_run": True}), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------ GPU arm
def parity_gate(Q, feats, res, pca_k):
    """Image 0 of this rank through the CPU oracle vs the GPU map (max-abs
    relative to max|ref| <= 1e-4); bins of image 0 bit-exact."""
    import numpy as np
    from oracle import qfca_oracle as O
    O.set_threads(os.cpu_count() or 1)
    x0 = feats[0].cpu().numpy()
    out = {"image": 0, "tol": 1e-4}
    if pca_k > 0:
        # QFCA+: score the GPU's own residual on the oracle (bins / R bit-exact by
        # construction of the protocol); the raw end-to-end
        # deviation is reported beside it (all-zero channels)
        import torch
        mean, comps, _ = Q.features.pca_fit_batch(feats[:1], min(pca_k, feats.shape[1]))
        r0 = Q.features.pca_residual_batch(feats[:1], mean, comps)[0].cpu().numpy()
        ref, img, _ = O.detect(r0)
        raw, _, _ = O.detect(x0, pca_components=pca_k)
        got = res.scores[0].cpu().numpy()
        out["protocol"] = "oracle fed the GPU residual"
        out["raw_e2e_rel_err"] = float(np.abs(got - raw).max() / np.abs(raw).max())
        del torch
    else:
        ref, img, _ = O.detect(x0)
        got = res.scores[0].cpu().numpy()
        lo, hi, dg = O.fit_quantizer(x0, 16)
        q = Q.fit_quantizer(feats[0], 16)
        bins = Q.bin_indices(feats[0], q).indices.cpu().numpy()
        out["bins_bit_exact"] = bool(np.array_equal(bins, O.bin_indices(x0, lo, hi, dg, 16)))
    out["max_rel_err"] = float(np.abs(got - ref).max() / np.abs(ref).max())
    out["image_score_abs_err"] = abs(float(res.image_scores[0]) - img)
    ok = out["max_rel_err"] <= 1e-4 and out.get("bins_bit_exact", True)
    out["pass"] = bool(ok)
    if not ok:
        raise AssertionError(f"parity gate failed on the bench workload: {out}")
    return out


def run_batch(args, ws, rank, local, config, size, pca_k, per_rank, mp_per_image):
    import numpy as np
    import torch
    import paper_2510_15602_b200 as Q
    from paper_2510_15602_b200 import _native
    import workloads

    dist = init_dist(ws, local, "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = Q.PipelineConfig(pca_components=pca_k)
    with torch.no_grad():
        parts = [workloads.make_features(min(CHUNK, per_rank - i), size,
                                         seed=1000 + 7919 * rank + i, device=dev)[0]
                 for i in range(0, per_rank, CHUNK)]
    feats = torch.cat(parts) if len(parts) > 1 else parts[0]
    del parts
    torch.cuda.synchronize()
    b, c, h, w = feats.shape
    chunks = [(i, min(i + CHUNK, b)) for i in range(0, b, CHUNK)]
    outs = [Q.scoring.DetectResult(
        scores=torch.empty((j - i, h, w), dtype=torch.float64, device=dev),
        image_scores=torch.empty((j - i,), dtype=torch.float64, device=dev),
        used=torch.empty((j - i,), dtype=torch.int32, device=dev),
        nonfinite=torch.zeros((1,), dtype=torch.int32, device=dev)) for i, j in chunks]
    ups = torch.empty((b, size, size), dtype=torch.float32, device=dev)

    def step(events=None):
        torch.cuda.nvtx.range_push("qfca_step")  # ncu --nvtx-include qfca_step/
        for k, (i, j) in enumerate(chunks):
            ev = None if events is None else events[k]
            res = Q.detect_batch(feats[i:j], cfg, out=outs[k], score_events=ev)
            Q.scoring.upsample_batch_into(res.scores, ups[i:j])
        torch.cuda.nvtx.range_pop()

    # correctness gate on this workload: image 0 against the CPU oracle
    step()
    torch.cuda.synchronize()
    if any(int(o.nonfinite[0]) for o in outs):
        raise AssertionError("non-finite features")
    parity = parity_gate(Q, feats, outs[0], pca_k) if rank == 0 else None

    # ---- device-resident timed region ("value"); inputs (>= 2 GiB) exceed L2
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    sev = [[(E(), E()) for _ in chunks] for _ in range(args.steps)]
    for row in sev:  # torch creates the cudaEvent handle lazily, on first record
        for a, z in row:
            a.record()
            z.record()
    start, end = E(), E()
    torch.cuda.synchronize()
    launches0 = _native.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        start.record()
        for i in range(args.steps):
            step(sev[i])
        end.record()
        torch.cuda.synchronize()
    launches = _native.launch_count() - launches0
    elapsed_ms = max_over_ranks(start.elapsed_time(end), dist, dev)
    score_ms_step = sum(a.elapsed_time(z) for row in sev for a, z in row) / args.steps
    score_ms_launch = score_ms_step / len(chunks)
    ms_per_step = elapsed_ms / args.steps
    total_images = b * ws * args.steps
    ips = total_images / (elapsed_ms / 1e3)

    # ---- end to end through the public streaming API with host buffers ("e2e")
    e2e = None
    if not args.no_e2e:
        # DetectPipeline: every batch is copied from pinned host memory, scored,
        # upsampled, and maps + upsampled maps + image scores come back; one
        # batch's copies overlap its neighbour's scoring.  A step = the rank's
        # images in batches of CHUNK.
        import psutil
        need = feats.numel() * 4
        if psutil.virtual_memory().available > 3 * need + (8 << 30):
            host = [feats[i:j].cpu().pin_memory() for i, j in chunks]
            host_note = "every image its own pinned host buffer"
        else:
            one = feats[:CHUNK].cpu().pin_memory()
            host = [one[: j - i] for i, j in chunks]
            host_note = "one pinned host batch reused (host RAM)"
        pipe = Q.DetectPipeline(cfg, upsample_to=(size, size))
        h2d = feats.numel() * 4
        d2h = b * h * w * 8 + b * 8 + b * size * size * 4
        for _ in pipe.run(host[:2] * 1):
            pass
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        e0, e1 = E(), E()
        e0.record()
        n_done = 0
        for r in pipe.run(host * args.steps):
            n_done += int(r.image_scores.numel())
        e1.record()
        torch.cuda.synchronize()
        assert n_done == b * args.steps
        e_ms = max_over_ranks(e0.elapsed_time(e1), dist, dev)
        e2e = {"value": total_images / (e_ms / 1e3), "unit": "images/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "mp_per_s": total_images / (e_ms / 1e3) * mp_per_image,
               "ms_per_step": e_ms / args.steps, "host_inputs": host_note,
               "api": "paper_2510_15602_b200.DetectPipeline (detect_batch per batch of "
                      f"{CHUNK}, upsample_to=({size},{size}))"}

    # ---- roofline of the dominant kernel (k_score), algorithmic bytes per launch
    peak, peak_src = peak_hbm()
    alg_launch = alg_bytes_per_image(size, pca_k > 0) * CHUNK
    achieved = alg_launch / (score_ms_launch / 1e3) / 1e9
    traffic, issue, kname = None, None, "k_score"
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.workload}.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj.get("dram_bytes_per_launch")
            kname = tj.get("kernel", kname)
            # K4 is issue-bound, not HBM-bound: its instruction-issue
            # utilisation from the same ncu capture is the kernel-quality figure
            issue = {"issue_active_frac": tj.get("issue_active_frac"), "ipc": tj.get("ipc"),
                     "ipc_peak": 4.0, "source": tj.get("source")}
        except Exception:
            traffic, issue = None, None
    alg_step = alg_bytes_per_image(size, pca_k > 0) * b
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
            "kernel": kname + " (fused histogram/transport/association/channel-sum)",
            "alg_bytes_per_launch": alg_launch, "images_per_launch": CHUNK,
            "kernel_ms_per_launch": score_ms_launch, "launches_per_step": len(chunks),
            "step_ms": ms_per_step, "kernel_share_of_step": score_ms_step / ms_per_step,
            "step_alg_bytes_frac": (alg_step / (ms_per_step / 1e3) / 1e9) / peak,
            "issue": issue}

    # ---- CPU baseline (rank 0, N = 1 only): the reference itself on host cores
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        ncores = os.cpu_count() or 1
        x_host = feats[:ncores].cpu().numpy()
        cpu, why = reference_cpu_baseline(x_host, pca_k, size)
        port = port_cpu_baseline(x_host[:2], pca_k, size, max_seconds=8.0)
        if cpu is None:
            cpu = port
            cpu["why_not_reference"] = why
        else:
            cpu["port"] = port

    if rank == 0:
        line = {"metric": METRIC, "value": ips, "unit": "images/s",
                "mp_per_s": ips * mp_per_image, "n_gpus": ws, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": config["scaling"], "vs_baseline": None,
                "dtype": "f32 features / u8 bins / i32 counts / f32+f64 errors",
                "data": "synthetic", "config": config, "roofline": roof,
                "cpu_baseline": cpu, "e2e": e2e, "parity": parity,
                "gpu_launches": launches, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_sharded_image(args, ws, rank, local, config, size, mp_per_image):
    """configs[4]: one image, channels sharded over the ranks (sharding.py); a
    step = score this rank's channel slice + one all-reduce of the (h*w + 1)
    channel-sum buffer + finalise (mean, Gaussian, image score)."""
    import numpy as np
    import torch
    import paper_2510_15602_b200 as Q
    from paper_2510_15602_b200 import _native, sharding
    import workloads
    dist = init_dist(ws, local, "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    with torch.no_grad():
        feats, _ = workloads.make_features(1, size, seed=1000, device=dev)
    c_all = feats.shape[1]
    c0, c1 = sharding.shard_range(c_all, ws, rank)
    x = feats[0, c0:c1].contiguous()
    h, w = x.shape[1:]
    del feats
    torch.cuda.empty_cache()
    cfg = Q.PipelineConfig()
    config.update({"channels": c_all, "channels_per_rank": c1 - c0, "feature_size": h,
                   "global_batch": 1, "images_per_gpu": None,
                   "parallelism": f"channel-sharded x{ws}, one all-reduce per image",
                   "l2": "inputs larger than L2 (features 2 GiB per image)"})

    def step(xx):
        torch.cuda.nvtx.range_push("qfca_step")
        out = sharding.detect_channel_sharded(xx, cfg)
        torch.cuda.nvtx.range_pop()
        return out

    for _ in range(max(3, args.warmup)):
        step(x)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    launches0 = _native.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            step(x)
        e1.record()
        torch.cuda.synchronize()
    launches = _native.launch_count() - launches0
    ms = max_over_ranks(e0.elapsed_time(e1), dist, dev)
    ms_per_step = ms / args.steps
    ips = 1e3 / ms_per_step

    e2e = None
    if not args.no_e2e:  # host slice in, map + image score out, every step
        xh = x.cpu().pin_memory()
        xd = torch.empty_like(x)
        for _ in range(2):
            xd.copy_(xh, non_blocking=True)
            m, _, _ = step(xd)
            m.cpu()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            xd.copy_(xh, non_blocking=True)
            m, _, _ = step(xd)
            m.cpu()
        f1.record()
        torch.cuda.synchronize()
        e_ms = max_over_ranks(f0.elapsed_time(f1), dist, dev)
        e2e = {"value": 1e3 * args.steps / e_ms, "unit": "images/s",
               "h2d_bytes_per_step": xh.numel() * 4, "d2h_bytes_per_step": h * w * 8,
               "mp_per_s": 1e3 * args.steps / e_ms * mp_per_image}

    peak, peak_src = peak_hbm()
    alg = alg_bytes_per_image(size, False)
    achieved = alg / (ms_per_step / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
            "kernel": "whole step (wide-plane tiles on the fused kernel + K3 + K1/K2 + "
                      "all-reduce + finalise)", "kernel_ms_per_launch": ms_per_step,
            "step_ms": ms_per_step, "kernel_share_of_step": 1.0,
            "step_alg_bytes_frac": achieved / peak}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        from baseline import refpool
        ncores = os.cpu_count() or 1
        sub = x[:ncores].cpu().numpy()[:, None]  # one channel per worker
        if refpool.available() is None:
            pool = refpool.ReferencePool(sub, 0, 1024)
            try:
                el, _ = pool.step()
            finally:
                pool.close()
            per_img = el * c_all / sub.shape[0]
            cpu = {"value": 1.0 / per_img, "unit": "images/s", "cores": pool.workers,
                   "kind": "reference",
                   "sample": f"{sub.shape[0]} of the {c_all} 1024x1024 channels, one per "
                             f"worker through qfca.detect ({el:.1f} s), extrapolated "
                             f"x{c_all / sub.shape[0]:.0f} (channels are independent)"}
        else:
            from oracle import qfca_oracle as O
            O.set_threads(ncores)
            t0 = time.perf_counter()
            O.detect(np.ascontiguousarray(x[:16].cpu().numpy()))
            el = time.perf_counter() - t0
            cpu = {"value": 16.0 / (el * c_all), "unit": "images/s", "cores": O.num_threads(),
                   "kind": "port", "sample": f"16 of {c_all} channels through the C oracle, "
                                              f"extrapolated", "why_not_reference":
                   refpool.available()}
    if rank == 0:
        line = {"metric": METRIC, "value": ips, "unit": "images/s",
                "mp_per_s": ips * mp_per_image, "n_gpus": ws, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32 features / u8 bins / i32 counts / f32+f64 errors",
                "data": "synthetic", "config": config, "roofline": roof, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0,
                    help="images (global for global workloads, else per GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="host stand-in for the GPU step, gloo backend (launch test)")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args.gpus))
    ws, rank, local = dist_env()
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; using {ws}", file=sys.stderr)

    size, images, is_global, pca_k, scaling, label = WORKLOADS[args.workload]
    images = args.batch or images
    mp_per_image = size * size / 1e6
    if is_global:
        from paper_2510_15602_b200.sharding import shard_range
        lo, hi = shard_range(images, ws, rank)
        per_rank = hi - lo
        global_batch = images
    else:
        per_rank, global_batch = images, images * ws
    config = {"workload": args.workload, "description": label, "global_batch": global_batch,
              "images_per_gpu": per_rank, "image_size": size, "channels": 512,
              "feature_size": size // 8, "n_bins": 16, "patch_size": 9,
              "pca_components": pca_k, "scaling": scaling,
              "parallelism": f"dp{ws} (images sharded, no comms)",
              "l2": "inputs larger than L2 (features >= 2 GiB per GPU)"}

    if args.dry_run:
        return run_dry(args, ws, rank, config, per_rank)
    if args.impl == "reference":
        return run_reference_arm(args, ws, rank, config, size, pca_k, mp_per_image)
    if args.workload == "qfca8192":
        return run_sharded_image(args, ws, rank, local, config, size, mp_per_image)
    return run_batch(args, ws, rank, local, config, size, pca_k, per_rank, mp_per_image)


if __name__ == "__main__":
    main()
