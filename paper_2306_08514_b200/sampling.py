"""Critical sampling of the TD GCCs on the GPU (batched real inverse FFT).

Drop-in for srpmap/sampling.py: `SampleSpec` (:31-65), `sample_spec` (:68-84),
`TdGccSamples` (:87-96) and `td_gcc_samples` (:106-134).  The GPU always uses
the iFFT path (the reference's "matrix" path agrees with it to <= 1e-12,
sampling.py:1-16, tests/test_sampling.py:81-88), so `path` only selects the
validation: "matrix" | "ifft" are accepted, anything else is a ValueError.

Output layout matches the reference: per frame the S = sum_p (2 N_p + 1) lags,
pair-major, each block in storage order 0..N_p, -N_p..-1.  Batched calls
return (F, S).  `frames_to_samples` is the fused signal -> samples chain.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dev
from . import _native as nat
from .errors import ConfigError, DimensionError
from .tiles import natural_columns as natural_source
from .frontend import (FdGcc, _check_range, _floor_args, _frame_range, _pairs_device, _signal,
                       _window_device, num_frames)


@dataclass(frozen=True)
class SampleSpec:
    counts: np.ndarray   # (P,) N_p
    n_aux: int
    half_len: int

    @property
    def num_pairs(self) -> int:
        return self.counts.shape[0]

    @property
    def samples_per_pair(self) -> np.ndarray:
        return 2 * self.counts + 1

    @property
    def total_samples(self) -> int:
        return int(np.sum(self.samples_per_pair))

    @property
    def mean_samples(self) -> float:
        return self.total_samples / self.num_pairs

    @property
    def offsets(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(self.samples_per_pair)])

    def lag_indices(self, p: int) -> np.ndarray:
        c = int(self.counts[p])
        return np.concatenate([np.arange(c + 1), np.arange(-c, 0)])


def spec_offsets(spec) -> np.ndarray:
    counts = np.asarray(spec.counts, dtype=np.int64)
    return np.concatenate([[0], np.cumsum(2 * counts + 1)]).astype(np.int64)


def sample_spec(tdoa, frame, n_aux: int = 2) -> SampleSpec:
    """N_p = floor(limit_p / T) + n_aux; ConfigError if 2 N_p + 1 > frame_len."""
    if n_aux < 0:
        raise ConfigError("n_aux must be non-negative")
    counts = np.floor(tdoa.limits / frame.sample_period).astype(np.int64) + n_aux
    worst = int(np.argmax(counts))
    if 2 * counts[worst] + 1 > frame.frame_len:
        raise ConfigError(f"frame length {frame.frame_len} too short: pair {worst} needs "
                          f"{2 * counts[worst] + 1} lag samples")
    return SampleSpec(counts=counts, n_aux=n_aux, half_len=frame.half_len)


@dataclass(frozen=True)
class TdGccSamples:
    """TD GCC samples: values (S,) or (F, S) float32 on the device.

    Kernels produce them lag-major: `lag_major` is the (S, ld) device buffer
    (frames contiguous, ld = F rounded up to 4) that the map kernels read, and
    `values` is its (F, S) view in the reference's per-frame layout.
    """

    values: torch.Tensor
    spec: object
    lag_major: object = field(default=None, repr=False, compare=False)
    # bf16 hi/lo planes for the tensor-core interpolation maps (optional): frame-major
    # [2][F][cols8] in storage order, or (planes_natural) lag-major [2][cols8][F8] with the
    # samples in natural lag order per pair
    bf16_planes: object = field(default=None, repr=False, compare=False)
    planes_natural: bool = field(default=False, repr=False, compare=False)
    # the planes are fp32 TF32 hi / lo (lag-major [2][cols8][F32], natural order) for the
    # 3xTF32 gathered-window engine instead of bf16
    planes_tf32: bool = field(default=False, repr=False, compare=False)
    # plane format: "bf16" | "tf32" | "f16" (fp16 hi / lo, lag-major [2][cols8][F64], natural
    # order: the fp16x3 gathered-window engine; PHAT samples only -- bounded by 2(K-1))
    planes_fmt: str = field(default="bf16", repr=False, compare=False)
    # produced with PHAT weighting by these kernels: |xi| <= 2(K-1), so fp16 operands are safe
    phat: bool = field(default=False, repr=False, compare=False)

    @property
    def num_frames(self) -> int:
        return 1 if self.values.dim() == 1 else self.values.shape[0]

    def per_pair(self, p: int) -> torch.Tensor:
        off = spec_offsets(self.spec)
        return self.values[..., off[p]:off[p + 1]]


def _spec_device(spec):
    def build():
        off = spec_offsets(spec)
        return dev.as_i32(np.asarray(spec.counts)), dev.as_i32(off)
    return dev.CACHE.get(spec, "spec_i32", build)


def pad4(n: int) -> int:
    return (int(n) + 3) // 4 * 4


def pad8(n: int) -> int:
    return (int(n) + 7) // 8 * 8


def _new_samples(frames: int, s_total: int, dev_):
    """Lag-major output buffer (S, ld) and its (F, S) view."""
    ld = pad4(max(frames, 1))
    buf = torch.empty((s_total, ld), dtype=torch.float32, device=dev_)
    return buf, ld, buf[:, :frames].t()


def _wrap(view, buf, spec, batched: bool, planes=None, natural: bool = False,
          fmt: str = "bf16", phat: bool = False) -> "TdGccSamples":
    return TdGccSamples(values=view if batched else view[0], spec=spec, lag_major=buf, bf16_planes=planes,
                        planes_natural=natural, planes_tf32=(fmt == "tf32"), planes_fmt=fmt, phat=phat)


def pad32(n: int) -> int:
    return (int(n) + 31) // 32 * 32


def pad64(n: int) -> int:
    return (int(n) + 63) // 64 * 64


def natural_source_device(spec):
    return dev.CACHE.get(spec, "natural_src_i32", lambda: dev.as_i32(natural_source(spec_offsets(spec))))


def _check_gcc(gcc, spec) -> None:
    if gcc.num_pairs != spec.num_pairs or gcc.num_bins != spec.half_len - 1:
        raise DimensionError(
            f"cross-spectra ({gcc.num_pairs} pairs x {gcc.num_bins} bins) do not match "
            f"sampling for {spec.num_pairs} pairs at K={spec.half_len}")


def td_gcc_samples(gcc, spec, path: str = "ifft") -> TdGccSamples:
    """Unnormalized real iDFT per pair, kept lags only (sampling.py:106-134)."""
    _check_gcc(gcc, spec)
    if path not in ("matrix", "ifft"):
        raise ValueError(f"unknown sampling path {path!r}")
    vals = dev.as_c64(gcc.values)
    batched = vals.dim() == 2
    vals = vals.reshape(-1, gcc.num_pairs * gcc.num_bins)
    counts, offsets = _spec_device(spec)
    s_total = int(spec_offsets(spec)[-1])
    buf, ld, view = _new_samples(vals.shape[0], s_total, vals.device)
    nat.call("srpgpu_td_gcc_samples", dev.ptr(vals), vals.shape[0], gcc.num_pairs, spec.half_len,
             dev.ptr(counts), dev.ptr(offsets), s_total, dev.ptr(buf), ld, dev.stream_ptr())
    return _wrap(view, buf, spec, batched)


def frames_to_samples(samples, frame, pairs, spec, frames=None, weighting: str = "phat",
                      floor=None, planes: bool = False, natural: bool = False,
                      tf32: bool = False, fmt: str | None = None) -> TdGccSamples:
    """Fused stft_frame -> fd_gcc -> td_gcc_samples for a range of frames.

    Neither the spectra nor the cross-spectra touch HBM; one kernel launch.  With
    `planes` the same kernel also writes the bf16 hi/lo planes the tensor-core
    interpolation maps read (`bf16_planes`; natural lag order per pair with `natural`,
    the layout of the gathered-window engine; with `tf32` (or fmt="tf32") too, fp32 TF32
    hi / lo planes for its 3xTF32 kernel; fmt="f16": fp16 hi / lo planes for its fp16x3
    kernel -- PHAT weighting only, whose samples are bounded by 2(K-1)).
    """
    fmt = fmt or ("tf32" if tf32 else "bf16")
    if fmt not in ("bf16", "tf32", "f16"):
        raise ValueError(f"unknown plane format {fmt!r}")
    if fmt != "bf16" and not natural:
        raise ValueError("TF32 / fp16 planes are natural-order lag-major only (natural=True)")
    if fmt == "f16" and planes and weighting != "phat":
        raise ValueError("fp16 planes need PHAT weighting (bounded samples); use fmt='tf32'")
    x = _signal(samples)
    if x.shape[0] != pairs.num_mics:
        raise DimensionError(f"expected {pairs.num_mics} channels, got {x.shape[0]}")
    if spec.num_pairs != pairs.num_pairs or spec.half_len != frame.half_len:
        raise DimensionError("sample spec does not match the pairs / frame")
    first, count, batched = _frame_range(frames, num_frames(frame, x.shape[1]))
    _check_range(frame, first, count, x.shape[1])
    w, mode, fval = _floor_args(weighting, floor)
    counts, offsets = _spec_device(spec)
    s_total = int(spec_offsets(spec)[-1])
    buf, ld, view = _new_samples(count, s_total, x.device)
    args = (dev.ptr(x), x.shape[0], x.shape[1], x.shape[1], dev.ptr(_window_device(frame)), frame.frame_len,
            frame.hop, first, count, dev.ptr(_pairs_device(pairs)), pairs.num_pairs, w, mode, fval,
            dev.ptr(counts), dev.ptr(offsets), s_total, dev.ptr(buf), ld)
    if not planes:
        nat.call("srpgpu_frames_to_samples", *args, dev.stream_ptr())
        return _wrap(view, buf, spec, batched, phat=(weighting == "phat"))
    cols8 = (s_total + 7) // 8 * 8
    src = natural_source_device(spec) if natural else None
    if fmt == "tf32":   # lag-major natural-order fp32 planes [2][cols8][F32] (3xTF32 gathered windows)
        planes_ld = pad32(count)
        pl = torch.empty((2, cols8, planes_ld), dtype=torch.float32, device=x.device)
    elif fmt == "f16":  # lag-major natural-order fp16 planes [2][cols8][F64] (fp16x3 gathered windows)
        planes_ld = pad64(count)
        pl = torch.empty((2, cols8, planes_ld), dtype=torch.float16, device=x.device)
    elif natural:   # lag-major natural-order planes [2][cols8][F8] (gathered-window engine)
        f8 = pad8(count)
        pl = torch.empty((2, cols8, f8), dtype=torch.bfloat16, device=x.device)
        planes_ld = f8
    else:           # frame-major planes [2][F][cols8] (dense tensor-core engine)
        pl = torch.empty((2, count, cols8), dtype=torch.bfloat16, device=x.device)
        planes_ld = 0
    nat.call("srpgpu_frames_to_samples_planes", *args, dev.ptr(pl), cols8, planes_ld,
             (1 if natural else 0) | (2 if fmt == "tf32" else 0) | (4 if fmt == "f16" else 0), dev.ptr(src),
             dev.stream_ptr())
    return _wrap(view, buf, spec, batched, pl, natural, fmt, phat=(weighting == "phat"))


def spectra_to_samples(spectra, pairs, spec, weighting: str = "phat", floor=None) -> TdGccSamples:
    """Fused fd_gcc -> td_gcc_samples on precomputed spectra (M, K+1) / (F, M, K+1)."""
    y = dev.as_c64(spectra)
    batched = y.dim() == 3
    if y.dim() == 2:
        y = y.unsqueeze(0)
    if y.dim() != 3 or y.shape[1] != pairs.num_mics or y.shape[2] != spec.half_len + 1:
        raise DimensionError(f"spectra of shape {tuple(y.shape)} do not match the pairs / spec")
    w, mode, fval = _floor_args(weighting, floor)
    counts, offsets = _spec_device(spec)
    s_total = int(spec_offsets(spec)[-1])
    buf, ld, view = _new_samples(y.shape[0], s_total, y.device)
    nat.call("srpgpu_spectra_to_samples", dev.ptr(y), y.shape[0], y.shape[1], spec.half_len,
             dev.ptr(_pairs_device(pairs)), pairs.num_pairs, w, mode, fval, dev.ptr(counts),
             dev.ptr(offsets), s_total, dev.ptr(buf), ld, dev.stream_ptr())
    return _wrap(view, buf, spec, batched, phat=(weighting == "phat"))


__all__ = ["SampleSpec", "TdGccSamples", "sample_spec", "td_gcc_samples", "frames_to_samples",
           "spectra_to_samples", "spec_offsets", "FdGcc"]
