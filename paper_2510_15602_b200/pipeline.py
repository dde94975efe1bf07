"""Streaming host -> device -> host driver around ``detect_batch``.

A serving loop feeds batches of features that live in host memory.  The
reference scores one image at a time on the CPU (scoring.py:235-299); on the
B200 the PCIe copy of a batch (C x H x W float32 per image) takes as long as
scoring it, so the driver overlaps them: batch i+1 is copied on a dedicated
copy stream into the second of two device buffers while batch i is scored on
the compute stream, and each batch's maps travel back into pinned host
buffers as soon as its scoring ends.  Events order the three engines; the
host blocks only when it reads a result.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Iterator

import torch

from .scoring import PipelineConfig, detect_batch, upsample_batch

__all__ = ["HostResult", "DetectPipeline"]


@dataclass
class HostResult:
    """One batch's results in pinned host memory.

    Lifetime: the tensors are views of the pipeline's two reusable pinned
    buffers.  They hold this batch's results until the caller asks the
    generator for the next result; after that the buffers are refilled by a
    later batch.  Clone them (or run with ``copy=True``) to keep them.
    """
    index: int
    scores: torch.Tensor          # (B, h, w) float64
    image_scores: torch.Tensor    # (B,) float64
    upsampled: torch.Tensor | None  # (B, H, W) float32 when ``upsample_to`` is set


class DetectPipeline:
    """Double-buffered streaming ``detect_batch`` for host-resident batches.

    ``run(batches)`` takes an iterable of (B, C, h, w) float32 CPU tensors
    (pinned for asynchronous copies; unpinned ones are staged through a
    pinned buffer) with one (C, h, w) and B no larger than the first batch's,
    and yields a ``HostResult`` per batch, in order (see HostResult for how
    long its tensors stay valid; ``copy=True`` yields owned copies).  ``upsample_to = (H, W)`` also returns the image-resolution maps
    (upsample_scores, scoring.py:149-152).
    """

    def __init__(self, cfg: PipelineConfig | None = None, upsample_to=None, device=None):
        self.cfg = cfg or PipelineConfig()
        self.upsample_to = upsample_to
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        self.copy_stream = torch.cuda.Stream(device=self.device)
        self.d2h_stream = torch.cuda.Stream(device=self.device)
        self._shape = None

    def _alloc(self, shape):
        b, c, h, w = shape
        dev = self.device
        self._shape = tuple(shape)
        self.dev_in = [torch.empty(shape, dtype=torch.float32, device=dev) for _ in range(2)]
        self.stage = [None, None]  # pinned staging for unpinned inputs, made on first use
        self.h_scores = [torch.empty((b, h, w), dtype=torch.float64).pin_memory()
                         for _ in range(2)]
        self.h_img = [torch.empty((b,), dtype=torch.float64).pin_memory() for _ in range(2)]
        self.h_up = None
        if self.upsample_to is not None:
            H, W = self.upsample_to
            self.h_up = [torch.empty((b, H, W), dtype=torch.float32).pin_memory()
                         for _ in range(2)]
        self.copied = [torch.cuda.Event() for _ in range(2)]    # input on the device
        self.freed = [torch.cuda.Event() for _ in range(2)]     # input buffer read
        self.done = [torch.cuda.Event() for _ in range(2)]      # results on the host

    def _copy_in(self, host: torch.Tensor, slot: int):
        n = host.shape[0]
        src = host
        if not host.is_pinned():
            if self.stage[slot] is None:
                self.stage[slot] = torch.empty(self._shape, dtype=torch.float32).pin_memory()
            self.copied[slot].synchronize()  # the staging buffer's last copy has been read
            self.stage[slot][:n].copy_(host)
            src = self.stage[slot][:n]
        with torch.cuda.stream(self.copy_stream):
            # the buffer is free once the compute that last read it has run
            self.copy_stream.wait_event(self.freed[slot])
            self.dev_in[slot][:n].copy_(src, non_blocking=True)
            self.copied[slot].record(self.copy_stream)

    def _check(self, batch: torch.Tensor):
        if (batch.dim() != 4 or tuple(batch.shape[1:]) != self._shape[1:]
                or batch.shape[0] > self._shape[0] or batch.shape[0] < 1):
            raise ValueError("every batch needs the first batch's (C, h, w) and at most "
                             "its number of images")

    def run(self, batches: Iterable[torch.Tensor], copy: bool = False) -> Iterator[HostResult]:
        it = iter(batches)
        try:
            first = next(it)
        except StopIteration:
            return
        if self._shape != tuple(first.shape):
            self._alloc(first.shape)
        compute = torch.cuda.current_stream(self.device)
        for ev in self.freed:
            ev.record(compute)
        self._copy_in(first, 0)
        pending = None  # (index, slot, images) whose results are in flight
        i, cur = 0, first
        while cur is not None:
            slot = i & 1
            n = cur.shape[0]
            nxt = next(it, None)
            if nxt is not None:
                self._check(nxt)
                self._copy_in(nxt, slot ^ 1)
            compute.wait_event(self.copied[slot])
            res = detect_batch(self.dev_in[slot][:n], self.cfg)
            self.freed[slot].record(compute)
            outs = [(res.scores, self.h_scores[slot][:n]),
                    (res.image_scores, self.h_img[slot][:n])]
            if self.h_up is not None:
                outs.append((upsample_batch(res.scores, *self.upsample_to),
                             self.h_up[slot][:n]))
            # results travel back on their own stream: the next batch's scoring
            # does not queue behind this batch's device -> host copies
            self.d2h_stream.wait_stream(compute)
            with torch.cuda.stream(self.d2h_stream):
                for dev_t, host_t in outs:
                    dev_t.record_stream(self.d2h_stream)
                    host_t.copy_(dev_t, non_blocking=True)
                self.done[slot].record(self.d2h_stream)
            if pending is not None:
                yield self._result(*pending, copy)
            pending = (i, slot, n)
            i, cur = i + 1, nxt
        if pending is not None:
            yield self._result(*pending, copy)

    def _result(self, index: int, slot: int, n: int, copy: bool) -> HostResult:
        self.done[slot].synchronize()
        up = None if self.h_up is None else self.h_up[slot][:n]
        r = HostResult(index=index, scores=self.h_scores[slot][:n],
                       image_scores=self.h_img[slot][:n], upsampled=up)
        if copy:
            r = HostResult(index=index, scores=r.scores.clone(),
                           image_scores=r.image_scores.clone(),
                           upsampled=None if up is None else up.clone())
        return r
