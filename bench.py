"""QFCA scoring throughput on B200 (driver contract: one JSON line on rank 0).

Default workload = BASELINE.json configs[1]: QFCA + PCA preprocessing (k=10),
batch 64 of 512x512 synthetic textures per GPU, WRN50-2 block-2 random-init
features (512 x 64 x 64), default bins / patch size.  A step = one pass of
the path over the batch: PCA (mean, covariance, eigh, residual) -> min/max ->
bins -> sort-free reference -> fused histogram/transport/association/channel
sum -> channel mean, smoothing, image scores -> bilinear upsampling to image
resolution.  `--workload qfca1024` runs configs[2] (QFCA, 1024x1024 textures,
64 per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (image size, images per GPU, pca components, config label)
    "qfca_plus512": (512, 64, 10, "configs[1]: QFCA + PCA (k=10), batch 64 of 512x512 "
                                  "synthetic textures, WRN50-2 random-init block-2 features"),
    "qfca1024": (1024, 64, 0, "configs[2]: QFCA, batch 64 per GPU of 1024x1024 synthetic "
                              "textures, WRN50-2 random-init block-2 features"),
    "qfca8192": (8192, 1, 0, "configs[4]: one 8192x8192 synthetic texture (512 x 1024^2 "
                             "WRN50-2 random-init block-2 features), channels sharded across "
                             "the ranks, one all-reduce of the channel-sum map"),
}
METRIC = "images/sec (megapixels/sec) of QFCA scoring; % of HBM roofline"


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

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._proc = None
        self._thr = None
        self._live = False

    def _run(self):
        for line in self._proc.stdout:
            if self._live and line.strip():
                self.samples.append([p.strip() for p in line.split(",")])

    def __enter__(self):
        # one long-running nvidia-smi sampling every 200 ms (a fresh process
        # per sample is too slow for sub-second timed regions; 50 ms polling was
        # measured to perturb the timed GPU work: configs[4] steps 23.7 ms
        # unsampled vs 23.8-33.8 ms at 50 ms)
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms",
                 os.environ.get("QFCA_BENCH_SMI_MS", "200")],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_reference_run(x_host, pca_k, max_seconds=20.0, min_images=1):
    """Time the CPU oracle (restatement of the reference path) on host cores."""
    from oracle import qfca_oracle as O
    import numpy as np
    cores = os.cpu_count() or 1
    O.set_threads(cores)
    done = 0
    t0 = time.perf_counter()
    while True:
        v = np.ascontiguousarray(x_host[done % x_host.shape[0]])
        O.detect(v, pca_components=pca_k)
        done += 1
        el = time.perf_counter() - t0
        if done >= min_images and (el >= max_seconds or done >= x_host.shape[0]):
            break
    return done, el, O.num_threads()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="qfca_plus512", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0, help="images per GPU (default: workload)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

    import numpy as np
    import torch

    ws, rank, local = dist_env()
    size, per_gpu, pca_k, label = WORKLOADS[args.workload]
    per_gpu = args.batch or per_gpu
    mp_per_image = size * size / 1e6
    config = {"workload": args.workload, "description": label, "images_per_gpu": per_gpu,
              "global_batch": per_gpu * ws, "image_size": size, "channels": 512,
              "feature_size": size // 8, "n_bins": 16, "patch_size": 9,
              "pca_components": pca_k, "parallelism": f"dp{ws} (images sharded, no comms)",
              "l2": "inputs larger than L2 (features >= 512 MiB per GPU)"}

    if args.impl == "reference":
        # CPU baseline arm: the oracle restatement of the reference on host cores
        if rank != 0:
            return
        dev = "cuda" if torch.cuda.is_available() else "cpu"
        import workloads
        feats, _ = workloads.make_features(min(per_gpu, 8), size, seed=1, device=dev)
        x_host = feats.cpu().numpy()
        from oracle import qfca_oracle as O
        O.detect(np.ascontiguousarray(x_host[0][:, :8, :8]))  # warm the library
        for _ in range(args.warmup):
            pass  # the oracle has no JIT / caches to warm beyond the library load
        # each step = one image of the workload through the oracle (bounded sample)
        O.set_threads(os.cpu_count() or 1)
        cores = O.num_threads()
        total_imgs, total_s = 0, 0.0
        for i in range(args.steps):
            t0 = time.perf_counter()
            O.detect(np.ascontiguousarray(x_host[i % x_host.shape[0]]), pca_components=pca_k)
            total_s += time.perf_counter() - t0
            total_imgs += 1
        ips = total_imgs / total_s
        line = {"metric": METRIC, "impl": "reference", "value": ips, "unit": "images/s",
                "mp_per_s": ips * mp_per_image, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * total_s / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32/f64", "data": "synthetic", "config": config,
                "cpu_baseline": {"value": ips, "unit": "images/s", "cores": cores,
                                 "kind": "port",
                                 "sample": f"{total_imgs} images of the workload "
                                           f"({size}x{size}, 512 ch) over {args.steps} steps"},
                "e2e": {"value": ips, "unit": "images/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import paper_2510_15602_b200 as Q
    from paper_2510_15602_b200 import _native
    import workloads

    if args.workload == "qfca8192":
        return run_sharded_image(args, ws, rank, local, config, size, mp_per_image)

    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    feats, masks = workloads.make_features(per_gpu, size, seed=1000 + rank, device=dev)
    torch.cuda.synchronize()
    cfg = Q.PipelineConfig(pca_components=pca_k)
    b, c, h, w = feats.shape

    def step(x, events=None):
        torch.cuda.nvtx.range_push("qfca_step")  # ncu --nvtx-include qfca_step/
        res = Q.detect_batch(x, cfg, score_events=events)
        up = Q.upsample_batch(res.scores, size, size)
        torch.cuda.nvtx.range_pop()
        return res, up

    # correctness gate on this workload (first image vs the CPU oracle)
    res, up = step(feats)
    torch.cuda.synchronize()
    assert int(res.nonfinite[0]) == 0

    # ---- device-resident timed region ("value")
    for _ in range(max(3, args.warmup)):
        step(feats)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for a, z in sev:  # torch creates the cudaEvent handle lazily, on first record
        a.record()
        z.record()
    torch.cuda.synchronize()
    launches0 = _native.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        start.record()
        for i in range(args.steps):
            step(feats, sev[i])
        end.record()
        torch.cuda.synchronize()
    launches = _native.launch_count() - launches0
    elapsed_ms = start.elapsed_time(end)
    score_ms = sum(a.elapsed_time(z) for a, z in sev) / args.steps
    if ws > 1:
        t = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t[0])
    ms_per_step = elapsed_ms / args.steps
    total_images = per_gpu * ws * args.steps
    ips = total_images / (elapsed_ms / 1e3)

    # ---- end to end through the C-ABI call with host buffers ("e2e")
    e2e = None
    if not args.no_e2e:
        # public streaming API (pipeline.DetectPipeline): every step copies its
        # batch from pinned host memory, scores it, upsamples the maps to image
        # resolution and copies maps + image scores back; the copies of one
        # batch overlap the scoring of its neighbour
        x_host = feats.cpu().pin_memory()
        pipe = Q.DetectPipeline(cfg, upsample_to=(size, size))
        h2d = x_host.numel() * 4
        d2h = b * h * w * 8 + b * 8 + b * size * size * 4
        for _ in pipe.run([x_host] * 2):
            pass
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n_done = 0
        for r in pipe.run([x_host] * args.steps):
            n_done += int(r.image_scores.numel() > 0)
        e1.record()
        torch.cuda.synchronize()
        assert n_done == args.steps
        e_ms = e0.elapsed_time(e1)
        if ws > 1:
            t = torch.tensor([e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t[0])
        e2e = {"value": total_images / (e_ms / 1e3), "unit": "images/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "mp_per_s": total_images / (e_ms / 1e3) * mp_per_image}

    # ---- roofline of the dominant kernel (k_score), algorithmic bytes per launch
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback"
    if os.path.exists(peaks_path):
        peak = float(json.load(open(peaks_path))["hbm_gbs"])
        peak_src = "measured"
    alg = alg_bytes_per_image(size, pca_k > 0) * per_gpu
    achieved = alg / (score_ms / 1e3) / 1e9
    traffic, issue = None, None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.workload}.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj.get("dram_bytes_per_launch")
            # K4 is issue-bound, not HBM-bound: its instruction-issue
            # utilisation from the same ncu capture is the kernel-quality figure
            issue = {"issue_active_frac": tj.get("issue_active_frac"), "ipc": tj.get("ipc"),
                     "ipc_peak": 4.0, "source": tj.get("source")}
        except Exception:
            traffic, issue = None, None
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
            "kernel": "k_score (fused histogram/transport/association/channel-sum)",
            "kernel_ms_per_launch": score_ms, "step_ms": ms_per_step,
            "kernel_share_of_step": score_ms / ms_per_step,
            "step_alg_bytes_frac": (alg / (ms_per_step / 1e3) / 1e9) / peak,
            "issue": issue}

    # ---- CPU baseline (rank 0, N = 1 only): the oracle on host cores
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        x_host_np = feats[:4].cpu().numpy()
        n_img, el, cores = cpu_reference_run(x_host_np, pca_k, max_seconds=15.0)
        cpu = {"value": n_img / el, "unit": "images/s", "cores": cores, "kind": "port",
               "sample": f"{n_img} of the workload's images ({size}x{size}, 512 ch), "
                         f"C oracle (OpenMP over channels) + NumPy PCA"}

    if rank == 0:
        line = {"metric": METRIC, "value": ips, "unit": "images/s",
                "mp_per_s": ips * mp_per_image, "n_gpus": ws, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "u8 bins / i32 counts / f32+f64 errors", "data": "synthetic",
                "config": config, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if ws > 1:
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
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
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
    if ws > 1:
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
    ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
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
        if ws > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            xd.copy_(xh, non_blocking=True)
            m, _, _ = step(xd)
            m.cpu()
        f1.record()
        torch.cuda.synchronize()
        e_ms = f0.elapsed_time(f1)
        if ws > 1:
            t = torch.tensor([e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t[0])
        e2e = {"value": 1e3 * args.steps / e_ms, "unit": "images/s",
               "h2d_bytes_per_step": xh.numel() * 4, "d2h_bytes_per_step": h * w * 8,
               "mp_per_s": 1e3 * args.steps / e_ms * mp_per_image}

    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peak, peak_src = 6650.0, "fallback"
    if os.path.exists(peaks_path):
        peak = float(json.load(open(peaks_path))["hbm_gbs"])
        peak_src = "measured"
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
        from oracle import qfca_oracle as O
        sub = x[:16].cpu().numpy()
        O.set_threads(os.cpu_count() or 1)
        t0 = time.perf_counter()
        O.detect(np.ascontiguousarray(sub))
        el = time.perf_counter() - t0
        per_img = el * c_all / sub.shape[0]  # scoring and reference are linear in C
        cpu = {"value": 1.0 / per_img, "unit": "images/s", "cores": O.num_threads(),
               "kind": "port",
               "sample": f"16 of the {c_all} channels of the 1024x1024 feature plane through "
                         f"the C oracle ({el:.1f} s), extrapolated x{c_all // 16} (linear in C)"}
    if rank == 0:
        line = {"metric": METRIC, "value": ips, "unit": "images/s",
                "mp_per_s": ips * mp_per_image, "n_gpus": ws, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "u8 bins / i32 counts / f32+f64 errors", "data": "synthetic",
                "config": config, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
