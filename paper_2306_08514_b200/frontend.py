"""Framing, STFT and pairwise cross-spectra with PHAT on the GPU.

Drop-in for the reference's srpmap/frontend.py: `FrameSpec` (:23-71),
`frame_window` (:74-79), `num_frames` (:82-86), `stft_frame` (:89-107),
`FdGcc` (:110-124) and `fd_gcc` (:127-160) keep their names, arguments and
error behaviour.  Every function additionally accepts a leading frame axis
(`frame_index` may be a range / slice / None for all frames), and results stay
on the device as torch tensors (complex64).  `gcc_frames` is the fused
samples -> cross-spectra entry (spectra never leave shared memory).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dev
from . import _native as nat
from .errors import DimensionError

PHAT_FLOOR_SCALE = 1e-12
WINDOWS = ("sqrt_hann", "rect", "hann")


@dataclass(frozen=True)
class FrameSpec:
    """Frame length 2K, sample rate, hop (default 2K/2), window.

    Windows: "sqrt_hann" (reference default), "rect" (reference test hook) and
    "hann" (periodic Hann, the BASELINE.json configs' window).
    """

    frame_len: int
    sample_rate: float
    hop: int = 0
    window: str = "sqrt_hann"

    def __post_init__(self):
        if self.frame_len < 4 or self.frame_len % 2 != 0:
            raise ValueError("frame_len must be even and >= 4")
        if not self.sample_rate > 0.0:
            raise ValueError("sample_rate must be positive")
        if self.hop == 0:
            object.__setattr__(self, "hop", self.frame_len // 2)
        if self.hop < 1:
            raise ValueError("hop must be >= 1")
        if self.window not in WINDOWS:
            raise ValueError(f"unknown window {self.window!r}")

    @property
    def half_len(self) -> int:
        return self.frame_len // 2

    @property
    def num_bins(self) -> int:
        return self.half_len - 1

    @property
    def sample_period(self) -> float:
        return 1.0 / self.sample_rate

    @property
    def bandlimit(self) -> float:
        return np.pi * self.sample_rate

    @property
    def bin_freqs(self) -> np.ndarray:
        return np.arange(1, self.half_len) * self.bandlimit / self.half_len


def frame_window(spec) -> np.ndarray:
    """Analysis window (float64, host)."""
    n = np.arange(spec.frame_len)
    window = getattr(spec, "window", "sqrt_hann")
    if window == "rect":
        return np.ones(spec.frame_len)
    if window == "hann":
        return 0.5 - 0.5 * np.cos(2.0 * np.pi * n / spec.frame_len)
    return np.sin(np.pi * n / spec.frame_len)


def num_frames(spec, num_samples: int) -> int:
    if num_samples < spec.frame_len:
        return 0
    return (num_samples - spec.frame_len) // spec.hop + 1


@dataclass(frozen=True)
class FdGcc:
    """Stacked cross-spectra at bins 1..K-1, pair-major: values (P*B,) or (F, P*B)."""

    values: torch.Tensor
    num_pairs: int
    num_bins: int
    weighting: str
    # set by gcc_frames(..., tf32=True): values rounded to TF32 (RNE), rows stored in
    # `padded` (F, ld) float32 with a 16-byte pitch, ready for the tensor-core map
    tf32_rounded: bool = field(default=False, compare=False)
    padded: object = field(default=None, repr=False, compare=False)

    @property
    def num_frames(self) -> int:
        return 1 if self.values.dim() == 1 else self.values.shape[0]

    def per_pair(self) -> torch.Tensor:
        if self.values.dim() == 1:
            return self.values.reshape(self.num_pairs, self.num_bins)
        return self.values.reshape(-1, self.num_pairs, self.num_bins)


_WINDOW_CACHE: dict = {}


def _window_device(spec) -> torch.Tensor:
    key = (spec.frame_len, getattr(spec, "window", "sqrt_hann"), torch.cuda.current_device())
    w = _WINDOW_CACHE.get(key)
    if w is None:
        w = dev.as_f32(frame_window(spec))
        _WINDOW_CACHE[key] = w
    return w


def _pairs_device(pairs) -> torch.Tensor:
    return dev.CACHE.get(pairs, "pairs_i32", lambda: dev.as_i32(np.asarray(pairs.pairs)))


def _frame_range(frame_index, total: int):
    """(first, count, batched) for an int, a unit-step range/slice, or None (all)."""
    if frame_index is None:
        return 0, total, True
    if isinstance(frame_index, slice):
        frame_index = range(*frame_index.indices(total))
    if isinstance(frame_index, range):
        if frame_index.step != 1 and len(frame_index) > 1:
            raise ValueError("frame ranges must have unit step")
        first = frame_index.start if len(frame_index) else 0
        return first, len(frame_index), True
    f = int(frame_index)
    return f, 1, False


def _signal(samples) -> torch.Tensor:
    x = dev.as_f32(samples)
    if x.dim() == 1:
        x = x.unsqueeze(0)
    if x.dim() != 2:
        raise DimensionError(f"samples must be (channels, num_samples), got {tuple(x.shape)}")
    return x


def _check_range(spec, first: int, count: int, num_samples: int) -> None:
    last = first + count - 1
    if count > 0 and (first < 0 or last * spec.hop + spec.frame_len > num_samples):
        bad = first if first < 0 else last
        raise IndexError(f"frame {bad} out of range for {num_samples} samples")


def stft_frame(samples, spec, frame_index) -> torch.Tensor:
    """Windowed DFT of frame(s): (M, K+1) or, batched, (F, M, K+1) complex64.

    frontend.py:89-107.  Frame f covers samples [f*hop, f*hop + frame_len).
    """
    x = _signal(samples)
    first, count, batched = _frame_range(frame_index, num_frames(spec, x.shape[1]))
    _check_range(spec, first, count, x.shape[1])
    m = x.shape[0]
    out = torch.empty((count, m, spec.half_len + 1), dtype=torch.complex64, device=x.device)
    nat.call("srpgpu_stft", dev.ptr(x), m, x.shape[1], x.shape[1], dev.ptr(_window_device(spec)),
             spec.frame_len, spec.hop, first, count, dev.ptr(out), None, dev.stream_ptr())
    return out if batched else out[0]


def _floor_args(weighting: str, floor):
    if weighting not in ("phat", "none"):
        raise ValueError(f"unknown weighting {weighting!r}")
    if floor is None:
        return (1 if weighting == "phat" else 0), 0, PHAT_FLOOR_SCALE
    return (1 if weighting == "phat" else 0), 1, float(floor)


def fd_gcc(spectra, pairs, weighting: str = "phat", floor=None) -> FdGcc:
    """Cross-spectra of all pairs at bins 1..K-1 with PHAT (frontend.py:127-160).

    spectra: (M, K+1) or (F, M, K+1).  floor: absolute PHAT floor; default
    1e-12 times the frame energy sum_{m,k} |Y|^2.
    """
    y = dev.as_c64(spectra)
    batched = y.dim() == 3
    if y.dim() == 2:
        y = y.unsqueeze(0)
    if y.dim() != 3 or y.shape[1] != pairs.num_mics:
        raise DimensionError(
            f"expected spectra for {pairs.num_mics} channels, got {tuple(np.shape(spectra))}")
    w, mode, fval = _floor_args(weighting, floor)
    bins = y.shape[2] - 2
    if bins < 1:
        raise DimensionError("spectra must cover at least bins 0..2")
    p = pairs.num_pairs
    out = torch.empty((y.shape[0], p * bins), dtype=torch.complex64, device=y.device)
    nat.call("srpgpu_fd_gcc", dev.ptr(y), y.shape[0], y.shape[1], bins + 1,
             dev.ptr(_pairs_device(pairs)), p, w, mode, fval, dev.ptr(out), dev.stream_ptr())
    return FdGcc(values=out if batched else out[0], num_pairs=p, num_bins=bins, weighting=weighting)


def gcc_frames(samples, spec, pairs, frames=None, weighting: str = "phat", floor=None,
               tf32: bool = False) -> FdGcc:
    """Fused stft_frame + fd_gcc over frames (default: all complete frames).

    tf32=True rounds the cross-spectra to TF32 (round-to-nearest-even) and pads
    rows to a 16-byte pitch: the operand layout of the tensor-core conventional map.
    """
    x = _signal(samples)
    if x.shape[0] != pairs.num_mics:
        raise DimensionError(f"expected {pairs.num_mics} channels, got {x.shape[0]}")
    first, count, batched = _frame_range(frames, num_frames(spec, x.shape[1]))
    _check_range(spec, first, count, x.shape[1])
    w, mode, fval = _floor_args(weighting, floor)
    p, bins = pairs.num_pairs, spec.num_bins
    ld = p * bins + ((p * bins) & 1 if tf32 else 0)          # complex elements per row
    buf = torch.empty((count, ld), dtype=torch.complex64, device=x.device)
    nat.call("srpgpu_gcc_frames", dev.ptr(x), x.shape[0], x.shape[1], x.shape[1],
             dev.ptr(_window_device(spec)), spec.frame_len, spec.hop, first, count,
             dev.ptr(_pairs_device(pairs)), p, w, mode, fval, dev.ptr(buf), ld, 1 if tf32 else 0,
             dev.stream_ptr())
    out = buf[:, :p * bins]
    padded = torch.view_as_real(buf).reshape(count, 2 * ld) if tf32 else None
    return FdGcc(values=out if batched else out[0], num_pairs=p, num_bins=bins, weighting=weighting,
                 tf32_rounded=tf32, padded=padded)


FRONTEND_KERNELS = {"auto": 0, "warp": 1, "task": 2, "block": 3}


class frontend_kernel:
    """Context manager selecting the frontend kernel (`srpgpu_set_frontend_kernel`).

    "auto" (default) picks by batch size; "warp" = a warp per frame
    (frontend_warp.cu), "task" = a warp per channel / pair task (frontend_lane.cu),
    "block" = the generic block kernel (frontend.cu).  All compute the same values;
    this is a tuning and testing knob.  Kernels captured in a CUDA graph keep the
    choice they were captured with.
    """

    def __init__(self, which: str):
        if which not in FRONTEND_KERNELS:
            raise ValueError(f"unknown frontend kernel {which!r}")
        self.which = which

    def __enter__(self):
        nat.call("srpgpu_set_frontend_kernel", FRONTEND_KERNELS[self.which])
        return self

    def __exit__(self, *exc):
        nat.call("srpgpu_set_frontend_kernel", 0)
