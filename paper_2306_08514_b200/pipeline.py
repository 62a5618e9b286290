"""Batched frames -> map -> argmax chains captured once as CUDA graphs.

The per-frame reference loop (cli.py:241-258: stft_frame -> fd_gcc ->
evaluate_map -> locate) becomes one graph replay per batch of frames:

    sspi / slri (latency-scale batches; sspi with short sparse rows): frames_to_sspi_map /
                       frames_to_slri_map -- the whole chain, argmax included, in one kernel
    sspi / si / slri :  frames_to_samples (1 fused kernel) -> map kernel(s) with fused argmax
    lr / conv        :  gcc_frames (1 fused kernel)        -> map kernel(s) with fused argmax

Replaying a captured graph removes the host launch latency that otherwise
dominates small batches (a 1000-frame cfg2 batch is ~10-50 us of GPU work).
The graph reads a static device input buffer and writes static outputs; `run`
copies a new batch in (from pinned host memory or device memory) and replays.
"""

from __future__ import annotations

import numpy as np
import torch

from . import maps, sampling
from . import frontend as fe
from ._device import device


class MapPipeline:
    """One captured CUDA graph for `frames` frames of `frame_len` samples."""

    VARIANTS = ("sspi", "si", "slri", "lr", "conv")

    def __init__(self, variant: str, op, frame, pairs, spec=None, frames: int = 1,
                 num_channels: int | None = None, weighting: str = "phat", floor=None,
                 out_map: bool = True, precision: str = "auto", graph: bool = True,
                 engine: str = "auto"):
        if variant == "conv_h":          # stored steering matrix: the same conventional chain
            variant = "conv"
        if variant not in self.VARIANTS:
            raise ValueError(f"unknown map variant {variant!r}")
        if variant in ("sspi", "si", "slri") and spec is None:
            raise ValueError(f"{variant} needs a SampleSpec")
        self.variant, self.op, self.frame, self.pairs, self.spec = variant, op, frame, pairs, spec
        self.frames = int(frames)
        self.weighting, self.floor, self.out_map = weighting, floor, out_map
        self.precision = maps.conv_precision(op, precision) if variant == "conv" else precision
        self.engine = engine              # sspi / si: "auto" | "fused" | "tc" | "tile" | "tile_f16" | "tile_bf16" | "band"
        m = num_channels or pairs.num_mics
        n = (self.frames - 1) * frame.hop + frame.frame_len
        self.input = torch.zeros((m, n), dtype=torch.float32, device=device())
        self.graph = None
        self._run_eager()                 # uploads operators, sets kernel attributes
        torch.cuda.synchronize()
        if graph:
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self.z, self.index = self._chain()
        else:
            self.z, self.index = self._run_eager()

    def _chain(self):
        rng = range(0, self.frames)
        v = self.variant
        if self.uses_fused_chain():
            # latency-scale batches: the whole chain in one kernel (xi never leaves shared memory)
            fused = maps.frames_to_sspi_map if v == "sspi" else maps.frames_to_slri_map
            return fused(self.op, self.input, self.frame, self.pairs, self.spec, rng,
                                           self.weighting, self.floor, argmax=True, out_map=self.out_map)
        if v in ("sspi", "si", "slri"):
            eng = maps.map_engine(v, self.op, self.engine, self.frames, bounded=maps.phat_bounded(self.weighting, self.frame.half_len))
            xi = sampling.frames_to_samples(self.input, self.frame, self.pairs, self.spec, rng,
                                            self.weighting, self.floor, **maps.plane_args(eng))
            if v == "slri":
                return maps.slri_map(self.op, xi, argmax=True, out_map=self.out_map)
            fn = maps.sspi_map if v == "sspi" else maps.si_map
            return fn(self.op, xi, argmax=True, out_map=self.out_map, engine=eng)
        gcc = fe.gcc_frames(self.input, self.frame, self.pairs, rng, self.weighting, self.floor,
                            tf32=(v == "conv" and self.precision == "tf32"))
        if v == "lr":
            return maps.lr_map(self.op, gcc, argmax=True, out_map=self.out_map)
        return maps.srp_map_exact(self.op, gcc, precision=self.precision, argmax=True,
                                  out_map=self.out_map)

    def uses_fused_chain(self) -> bool:
        """Latency-scale sspi / slri batches: the whole chain in one kernel
        (frames_to_sspi_map for short sparse rows, frames_to_slri_map)."""
        if self.variant not in ("sspi", "slri") or self.engine not in ("auto", "fused"):
            return False
        m = self.input.shape[0]
        if self.variant == "sspi":
            ok = maps.fused_eligible(self.op, self.frame, self.spec, self.frames, m)
            auto = ok
        else:
            ok = maps.fused_slri_eligible(self.op, self.frame, self.spec, self.frames, m)
            auto = ok and self.frames * np.asarray(self.op.tall).shape[0] < maps.LOWRANK_TC_MIN_OUTPUTS
        if self.engine == "fused":
            if not ok:
                raise ValueError(f"the fused {self.variant} chain does not take this operator / frame shape / batch")
            return True
        return auto

    def _run_eager(self):
        return self._chain()

    def replay(self):
        """Run the chain on the current contents of `self.input`."""
        if self.graph is not None:
            self.graph.replay()
            return self.z, self.index
        self.z, self.index = self._chain()
        return self.z, self.index

    def run(self, samples=None):
        """Copy a batch of samples (M, n) in (host pinned / device / numpy) and run."""
        if samples is not None:
            if isinstance(samples, np.ndarray):
                samples = torch.from_numpy(np.ascontiguousarray(samples, dtype=np.float32))
            self.input.copy_(samples, non_blocking=True)
        return self.replay()


class MapStream:
    """Streamed batches: host samples in, per-frame argmax out, copies overlapped.

    The batched counterpart of the reference's per-frame `cmd_map` loop
    (cli.py:241-258).  `depth` MapPipeline slots (each its own input buffer,
    graph and outputs) rotate; batch n's host->device copy runs on a copy
    stream while batch n-1's chain runs on the compute stream, and the per-frame
    argmax of each batch is read back into pinned host memory.  `after_batch`
    (e.g. an NCCL gather of argmax keys) is enqueued on the compute stream after
    each chain.
    """

    def __init__(self, variant: str, op, frame, pairs, spec=None, frames: int = 1, depth: int = 2,
                 after_batch=None, **kw):
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.slots = [MapPipeline(variant, op, frame, pairs, spec, frames=frames, **kw)
                      for _ in range(depth)]
        self.copy_stream = torch.cuda.Stream()
        self.compute_stream = torch.cuda.Stream()
        self.after_batch = after_batch
        self.frames = int(frames)
        self._out = [torch.empty(self.frames, dtype=torch.int64).pin_memory() for _ in range(depth)]
        self._free = [torch.cuda.Event() for _ in range(depth)]     # slot's chain has consumed its input
        self._done = [torch.cuda.Event() for _ in range(depth)]     # slot's argmax is on the host
        self._used = [False] * depth
        self._count = 0

    @property
    def input_shape(self):
        return tuple(self.slots[0].input.shape)

    def submit(self, samples) -> int:
        """Enqueue one batch of (M, n) samples (pinned host tensor for async copies)."""
        k = self._count % len(self.slots)
        slot = self.slots[k]
        if isinstance(samples, np.ndarray):
            samples = torch.from_numpy(np.ascontiguousarray(samples, dtype=np.float32))
        if tuple(samples.shape) != self.input_shape:
            raise ValueError(f"batch shape {tuple(samples.shape)} != {self.input_shape}")
        if self._used[k]:
            self._done[k].synchronize()    # the host may still be reading this slot's output
        cur = torch.cuda.current_stream()
        self.copy_stream.wait_stream(cur)
        with torch.cuda.stream(self.copy_stream):
            if self._used[k]:
                self.copy_stream.wait_event(self._free[k])
            slot.input.copy_(samples, non_blocking=True)
        self.compute_stream.wait_stream(self.copy_stream)
        with torch.cuda.stream(self.compute_stream):
            z, idx = slot.replay()
            self._free[k].record()
            if self.after_batch is not None:
                self.after_batch(idx)
            self._out[k].copy_(idx, non_blocking=True)
            self._done[k].record()
        self._used[k] = True
        self._count += 1
        return self._count - 1

    def result(self, ticket: int) -> np.ndarray:
        """Per-frame argmax of batch `ticket` (waits for it; valid until the slot is reused)."""
        if ticket < self._count - len(self.slots) or ticket >= self._count:
            raise ValueError(f"batch {ticket} is no longer (or not yet) held")
        k = ticket % len(self.slots)
        self._done[k].synchronize()
        return self._out[k].numpy().copy()

    def join(self):
        """Make the caller's current stream wait for every submitted batch."""
        torch.cuda.current_stream().wait_stream(self.compute_stream)
