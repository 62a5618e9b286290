"""Seeded synthetic scenes for the BASELINE.json configurations.

BASELINE.json names synthetic signals (white-Gaussian sources, white noise,
plane waves); the reference simulator only renders pink/WAV point sources
(simulate.py:151-265), so inputs come from this generator and the parity
boundary starts at the multichannel samples.
Propagation delays are applied exactly in the frequency domain (circular
fractional delay of a padded white sequence), with 1/r gain for near-field
sources and independent white noise at the configured SNR relative to the mean
direct-path power (the SNR rule of simulate.py:256-264).

    cfg1  NF 2D, M=4 in a 0.5 m square, J=41x41=1681, K=512, Hann, F=100
    cfg2  cfg1 geometry, F=1000 (LR / SLRI / SSPI sweeps)
    cfg3  FF 3D, UCA M=8 r=5 cm, 360 x 91 directions (J=32760), K=256, F=1e4
    cfg4  NF 3D, M=16 in a 1x1x0.5 m box, 5 cm grid 81x81x51 (J=334611), K=512, F=1e4
    cfg5  cfg3 geometry with a variable frame count
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .frontend import FrameSpec
from .sampling import sample_spec
from .scene import (MicrophoneArray, build_ff_grid, build_nf_grid, enumerate_pairs, tdoa_table)

C_SOUND = 343.0
FS = 16000.0


@dataclass
class Workload:
    name: str
    frame: FrameSpec
    array: MicrophoneArray
    pairs: object
    grid: object
    tdoa: object
    spec: object
    samples: np.ndarray          # (M, N) float32
    num_frames: int
    truth: np.ndarray            # (n_src, 3) positions (NF) or propagation directions (FF)
    info: dict = field(default_factory=dict)

    @property
    def num_candidates(self) -> int:
        return self.grid.num_points


def _delay_signals(rng, delays_s, gains, n: int, fs: float) -> np.ndarray:
    """x_m[t] = gain_m * s(t - delay_m) for one white source, exact fractional delay."""
    pad = 1 << int(np.ceil(np.log2(n + 4096)))
    s = rng.standard_normal(pad)
    spec = np.fft.rfft(s)
    w = 2.0 * np.pi * np.fft.rfftfreq(pad)          # rad / sample
    out = np.empty((len(delays_s), n))
    for m, (d, g) in enumerate(zip(delays_s, gains)):
        out[m] = g * np.fft.irfft(spec * np.exp(-1j * w * d * fs), n=pad)[2048:2048 + n]
    return out


def _add_noise(rng, direct: np.ndarray, snr_db: float) -> np.ndarray:
    power = float(np.mean(np.var(direct, axis=1)))
    sigma = np.sqrt(power / 10.0 ** (snr_db / 10.0))
    return direct + sigma * rng.standard_normal(direct.shape)


def _finish(name, frame, array, grid, samples, num_frames, truth, info) -> Workload:
    pairs = enumerate_pairs(array)
    tdoa = tdoa_table(array, pairs, grid)
    spec = sample_spec(tdoa, frame, 2)
    return Workload(name, frame, array, pairs, grid, tdoa, spec,
                    np.ascontiguousarray(samples, dtype=np.float32), num_frames, truth, info)


def nf2d(name: str, num_frames: int, seed: int = 1) -> Workload:
    """cfg1 / cfg2."""
    rng = np.random.default_rng([seed, 1])
    mics = np.column_stack([rng.uniform(1.75, 2.25, 4), rng.uniform(1.75, 2.25, 4), np.zeros(4)])
    array = MicrophoneArray(mics, C_SOUND)
    frame = FrameSpec(frame_len=1024, sample_rate=FS, hop=512, window="hann")
    grid = build_nf_grid((0, 0, 0), (4, 4, 0), 0.1)
    while True:
        src = np.array([rng.uniform(0, 4), rng.uniform(0, 4), 0.0])
        if np.min(np.linalg.norm(mics - src, axis=1)) >= 0.05:
            break
    n = (num_frames - 1) * frame.hop + frame.frame_len
    r = np.linalg.norm(mics - src, axis=1)
    direct = _delay_signals(rng, r / C_SOUND, 1.0 / r, n, FS)
    samples = _add_noise(rng, direct, 20.0)
    return _finish(name, frame, array, grid, samples, num_frames, src[None, :],
                   {"snr_db": 20.0, "mode": "nf"})


def ff3d(name: str, num_frames: int, seed: int = 3) -> Workload:
    """cfg3 / cfg5: UCA M=8, r = 5 cm, 1-3 plane waves, 10 dB."""
    rng = np.random.default_rng([seed, 3])
    array = MicrophoneArray.circular((0.0, 0.0, 0.0), 0.05, 8, C_SOUND)
    frame = FrameSpec(frame_len=512, sample_rate=FS, hop=256, window="hann")
    grid = build_ff_grid(1.0, collapse_poles=False)          # 91 x 360 = 32760
    n_src = int(rng.integers(1, 4))
    idx = rng.choice(grid.num_points, size=n_src, replace=False)
    dirs = grid.points[idx]
    n = (num_frames - 1) * frame.hop + frame.frame_len
    direct = np.zeros((array.num_mics, n))
    for q in dirs:
        delays = array.positions @ q / C_SOUND + 0.01        # bulk offset keeps delays positive
        direct += _delay_signals(rng, delays, np.ones(array.num_mics), n, FS)
    samples = _add_noise(rng, direct, 10.0)
    return _finish(name, frame, array, grid, samples, num_frames, dirs,
                   {"snr_db": 10.0, "mode": "ff", "sources": n_src, "source_index": idx})


def nf3d(name: str, num_frames: int, seed: int = 4) -> Workload:
    """cfg4: M=16 in a 1 x 1 x 0.5 m box centred in a 4 x 4 x 2.5 m room, 5 cm grid."""
    rng = np.random.default_rng([seed, 4])
    mics = np.column_stack([rng.uniform(1.5, 2.5, 16), rng.uniform(1.5, 2.5, 16),
                            rng.uniform(1.0, 1.5, 16)])
    array = MicrophoneArray(mics, C_SOUND)
    frame = FrameSpec(frame_len=1024, sample_rate=FS, hop=512, window="hann")
    grid = build_nf_grid((0, 0, 0), (4, 4, 2.5), 0.05)
    while True:
        src = rng.uniform([0, 0, 0], [4, 4, 2.5])
        if np.min(np.linalg.norm(mics - src, axis=1)) >= 0.05:
            break
    n = (num_frames - 1) * frame.hop + frame.frame_len
    r = np.linalg.norm(mics - src, axis=1)
    direct = _delay_signals(rng, r / C_SOUND, 1.0 / r, n, FS)
    samples = _add_noise(rng, direct, 20.0)
    return _finish(name, frame, array, grid, samples, num_frames, src[None, :],
                   {"snr_db": 20.0, "mode": "nf", "snr_assumed": True})


def make(cfg: str, num_frames: int | None = None, seed: int | None = None) -> Workload:
    kw = {} if seed is None else {"seed": seed}
    if cfg == "cfg1":
        return nf2d("cfg1", num_frames or 100, **kw)
    if cfg == "cfg2":
        return nf2d("cfg2", num_frames or 1000, **kw)
    if cfg == "cfg3":
        return ff3d("cfg3", num_frames or 10000, **kw)
    if cfg == "cfg4":
        return nf3d("cfg4", num_frames or 10000, **kw)
    if cfg == "cfg5":
        return ff3d("cfg5", num_frames or 1024, **kw)
    raise ValueError(f"unknown config {cfg!r}")
