"""Batched `map` command: a recording -> per-frame maps and locations.

The reference's `cmd_map` (cli.py:210-259) checks the operator cache against the
run configuration, loads the recording (frontend.py:163-185) and then, frame by
frame, runs STFT -> GCC -> map and writes one CSV row per candidate plus a
`summary` row with the map maximum (`locate`, srp.py:74-80; scored against a true
location with metrics.py:164-206 when given).  At J = 32760 the CSV writer alone
costs ~228 ms per frame [SURVEY §8(f)].

Here the whole recording runs as batched CUDA-graph chains (`MapPipeline`: one
frontend kernel and one map kernel with the fused argmax per batch); the maximum
and its value are gathered on the GPU, and only the summary rows are formatted on
the host unless the per-candidate maps are asked for -- as the reference's CSV rows
(`maps="csv"`, same format) or as a binary float32 `[frames][J]` array
(`maps="npy"`).  Row formatting follows cli.py:38-43 (`format(v, ".17g")`).

`read_run_config` reads the sections of the reference's INI run configuration
that `map` needs (config.py:1-33, 126-232) so that `params_hash` reproduces the
digest stored in the cache.
"""

from __future__ import annotations

import configparser
import csv
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import cache as _cache
from .errors import ConfigError
from .frontend import FrameSpec, num_frames
from .pipeline import MapPipeline
from .scene import MicrophoneArray, build_ff_grid, build_nf_grid, enumerate_pairs

NF_THRESHOLD = 0.2                      # metrics.py:35
FF_THRESHOLD = math.radians(2.5)        # metrics.py:38
STEEPNESS = 6.0                         # metrics.py:41
CSV_HEADER = ["row_type", "frame", "index", "qx", "qy", "qz", "value", "loc_error", "accuracy"]


# ------------------------------------------------------------------ inputs

def load_audio(path: str, sample_rate: float | None = None, channels: int | None = None):
    """(channels, samples) float32 and the sample rate (frontend.py:163-185).

    WAV 16-bit PCM is scaled by 1/32768 and 32-bit float is taken as is (both exact
    in float32, the kernels' input type); headerless .f32/.raw files are interleaved
    little-endian float32 and need `sample_rate` and `channels`.
    """
    path = str(path)
    if path.endswith((".f32", ".raw")):
        if sample_rate is None or channels is None:
            raise ValueError("raw float32 input needs sample_rate and channels")
        flat = np.fromfile(path, dtype="<f4")
        if flat.size % channels:
            raise ValueError(f"raw file length not divisible by {channels} channels")
        return np.ascontiguousarray(flat.reshape(-1, channels).T), float(sample_rate)
    from scipy.io import wavfile
    rate, data = wavfile.read(path)
    if data.dtype == np.int16:
        data = data.astype(np.float32) / np.float32(32768.0)
    else:
        data = data.astype(np.float32)
    if data.ndim == 1:
        data = data[:, None]
    return np.ascontiguousarray(data.T), float(rate)


@dataclass(frozen=True)
class RunScene:
    """What `map` needs from the run configuration (config.py:159-232)."""

    mode: str
    room: np.ndarray
    array: MicrophoneArray
    grid: object
    frame: FrameSpec
    weighting: str = "phat"
    n_aux: int = 2


def _nums(text: str, count: int | None = None) -> np.ndarray:
    try:
        v = np.array([float(t) for t in text.split()])
    except ValueError as exc:
        raise ConfigError(f"cannot parse number list {text!r}") from exc
    if count is not None and v.size != count:
        raise ConfigError(f"expected {count} numbers, got {text!r}")
    return v


def read_run_config(path: str) -> RunScene:
    """The scene/pipeline sections of a reference INI run configuration."""
    cp = configparser.ConfigParser(inline_comment_prefixes=(";", "#"))
    try:
        if not cp.read(path):
            raise ConfigError(f"cannot read config file {path!r}")
    except configparser.Error as exc:
        raise ConfigError(f"malformed config file {path!r}: {exc}") from exc
    for sec in ("scenario", "array", "grid", "pipeline"):
        if sec not in cp:
            raise ConfigError(f"missing [{sec}] section")
    sc, ar, gr, pl = cp["scenario"], cp["array"], cp["grid"], cp["pipeline"]
    mode = sc.get("mode", "")
    if mode not in ("nf", "ff"):
        raise ConfigError(f"scenario.mode must be nf or ff, got {mode!r}")
    c = float(ar.get("speed_of_sound", "343"))
    if ar.get("kind", "positions") == "circular":
        array = MicrophoneArray.circular(_nums(ar["center"], 3), float(ar["radius"]), int(ar["count"]), c)
    else:
        rows = [_nums(r, 3) for r in ar.get("positions", "").split(";") if r.strip()]
        if not rows:
            raise ConfigError("array.positions is empty")
        array = MicrophoneArray(np.vstack(rows), c)
    if mode == "nf":
        grid = build_nf_grid(_nums(gr["origin"], 3), _nums(gr["extents"], 3), float(gr["resolution"]))
    else:
        grid = build_ff_grid(float(gr["resolution_deg"]),
                             polar_deg=tuple(_nums(gr.get("polar_deg", "90 180"), 2)),
                             azimuth_deg=tuple(_nums(gr.get("azimuth_deg", "0 360"), 2)))
    frame = FrameSpec(frame_len=int(pl["frame_len"]), sample_rate=float(pl["sample_rate"]),
                      hop=int(pl.get("hop", "0")))
    weighting = pl.get("weighting", "phat")
    if weighting not in ("phat", "none"):
        raise ConfigError(f"weighting must be phat or none, got {weighting!r}")
    return RunScene(mode=mode, room=_nums(sc.get("room", ""), 3), array=array, grid=grid, frame=frame,
                    weighting=weighting, n_aux=int(pl.get("n_aux", "2")))


def scene_hash(scene: RunScene, kind: str, meta: dict) -> str:
    """params_hash of a cache built for this scene (cli.py:46-66, 213-218)."""
    return _cache.params_hash(mode=scene.mode, room=scene.room, positions=scene.array.positions,
                              speed_of_sound=scene.array.speed_of_sound, grid_axes=scene.grid.axes,
                              frame_len=scene.frame.frame_len, sample_rate=scene.frame.sample_rate,
                              hop=scene.frame.hop, weighting=scene.weighting, n_aux=scene.n_aux,
                              method=kind, rank=meta.get("rank"), keep=meta.get("keep"),
                              path=meta.get("path", "auto"))


# ------------------------------------------------------------------ the batched map

@dataclass
class RecordingMaps:
    index: np.ndarray            # (F,) argmax candidate (np.argmax tie rule)
    value: np.ndarray            # (F,) float32 map value there
    maps: np.ndarray | None      # (F, J) float32 when requested


def map_recording(kind: str, op, spec, frame: FrameSpec, pairs, samples, *, weighting: str = "phat",
                  batch_frames: int = 4096, keep_maps: bool = False) -> RecordingMaps:
    """Every complete frame of `samples` (M, N) through one batched chain per batch."""
    samples = np.ascontiguousarray(samples, dtype=np.float32)
    total = num_frames(frame, samples.shape[1])
    j = _num_candidates(kind, op)
    if total == 0:
        return RecordingMaps(np.zeros(0, np.int64), np.zeros(0, np.float32),
                             np.zeros((0, j), np.float32) if keep_maps else None)
    b = max(1, min(int(batch_frames), total))
    nb = (total + b - 1) // b
    need = (nb * b - 1) * frame.hop + frame.frame_len          # zero tail: padded frames are dropped
    host = torch.zeros((samples.shape[0], max(need, samples.shape[1])), dtype=torch.float32)
    host[:, :samples.shape[1]] = torch.from_numpy(samples)
    host = host.pin_memory()                                   # one pinned copy: async batch uploads
    variant = {"conv": "conv"}.get(kind, kind)
    pipe = MapPipeline(variant, op, frame, pairs, spec, frames=b, weighting=weighting)
    index = torch.empty(nb * b, dtype=torch.int64, device=pipe.input.device)
    value = torch.empty(nb * b, dtype=torch.float32, device=pipe.input.device)
    maps = np.empty((total, j), np.float32) if keep_maps else None
    for k in range(nb):
        x = host[:, k * b * frame.hop:k * b * frame.hop + pipe.input.shape[1]]
        z, idx = pipe.run(x)
        index[k * b:(k + 1) * b] = idx
        value[k * b:(k + 1) * b] = z.gather(1, idx[:, None])[:, 0]
        if keep_maps:
            m = min(b, total - k * b)
            maps[k * b:k * b + m] = z[:m].cpu().numpy()
    return RecordingMaps(index[:total].cpu().numpy(), value[:total].cpu().numpy(), maps)


def _num_candidates(kind, op) -> int:
    if kind in ("conv",):
        return int(op.matrix.shape[0]) if hasattr(op, "matrix") else int(op.num_candidates)
    if kind == "lr":
        return int(op.tall.shape[0])
    if kind == "si":
        return int(op.matrix.shape[0])
    if kind == "slri":
        return int(op.tall.shape[0])
    return int(np.asarray(op.row_splits).shape[0] - 1)


# ------------------------------------------------------------------ scoring and rows

def fmt(value) -> str:
    """cli.py:38-43."""
    if isinstance(value, float):
        if math.isinf(value):
            return "-inf" if value < 0 else "inf"
        return format(value, ".17g")
    return str(value)


def loc_error(estimate, truth, mode: str) -> float:
    """metrics.py:164-172: metres (nf) or radians (ff)."""
    e, t = np.asarray(estimate, dtype=float), np.asarray(truth, dtype=float)
    if mode == "nf":
        return float(np.linalg.norm(e - t))
    if mode == "ff":
        return float(math.acos(min(1.0, max(-1.0, float(e @ t)))))
    raise ValueError(f"unknown mode {mode!r}")


def loc_accuracy(error: float, threshold: float, steepness: float = STEEPNESS) -> float:
    """metrics.py:175-181: sigmoid score, 0.5 at the threshold."""
    if not threshold > 0.0:
        raise ValueError("threshold must be positive")
    arg = min(700.0, max(-700.0, steepness * (error - threshold) / threshold))
    return 1.0 / (1.0 + math.exp(arg))


def parse_truth(text: str, scene: RunScene) -> np.ndarray:
    """cli.py:200-207 (ff truths given as a position become the incident direction)."""
    vals = np.array([float(t) for t in text.replace(",", " ").split()])
    if vals.shape != (3,):
        raise ConfigError("--truth needs three numbers")
    if scene.mode == "ff" and abs(np.linalg.norm(vals) - 1.0) > 1e-6:
        d = scene.array.center - vals       # incident direction, source -> array (simulate.py:126-135)
        return d / np.linalg.norm(d)
    return vals


def write_map_csv(path: str, grid, result: RecordingMaps, truth=None, *, map_rows: bool = False) -> None:
    """The reference's map CSV (cli.py:236-258): optional per-candidate rows, one summary per frame."""
    pts = np.asarray(grid.points, dtype=float)
    thr = NF_THRESHOLD if grid.mode == "nf" else FF_THRESHOLD
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(CSV_HEADER)
        coords = [[fmt(float(v)) for v in q] for q in pts] if map_rows else None
        for f in range(result.index.shape[0]):
            if map_rows:
                zf = result.maps[f].astype(np.float64)
                for i in range(pts.shape[0]):
                    w.writerow(["map", f, i, *coords[i], fmt(float(zf[i])), "", ""])
            i = int(result.index[f])
            q = pts[i]
            err = acc = ""
            if truth is not None:
                e = loc_error(q, truth, grid.mode)
                err, acc = fmt(e), fmt(loc_accuracy(e, thr))
            w.writerow(["summary", f, i, fmt(float(q[0])), fmt(float(q[1])), fmt(float(q[2])),
                        fmt(float(result.value[f])), err, acc])


def cmd_map(scene: RunScene, cache_path: str, audio_path: str, out_path: str, truth_text: str | None = None,
            *, maps: str = "none", batch_frames: int = 4096) -> RecordingMaps:
    """cmd_map (cli.py:210-259) on the GPU: maps = "none" | "csv" | "npy"."""
    if maps not in ("none", "csv", "npy"):
        raise ValueError(f"maps must be none, csv or npy, got {maps!r}")
    bundle = _cache.load_cache(cache_path)
    if scene_hash(scene, bundle.kind, bundle.meta) != bundle.params_hash:
        raise ConfigError("cache/config mismatch: the cache was built for a different "
                          "scene, pipeline, or method; refusing to run")
    op, spec = _cache.operator_from_bundle(bundle)
    samples, rate = load_audio(audio_path, sample_rate=scene.frame.sample_rate,
                               channels=scene.array.num_mics)
    if abs(rate - scene.frame.sample_rate) > 1e-6:
        raise ConfigError(f"audio rate {rate} does not match configured {scene.frame.sample_rate}")
    if samples.shape[0] != scene.array.num_mics:
        raise ConfigError(f"audio has {samples.shape[0]} channels, array has {scene.array.num_mics}")
    truth = parse_truth(truth_text, scene) if truth_text else None
    _cache.upload(bundle.kind, op, spec)
    pairs = enumerate_pairs(scene.array)
    res = map_recording(bundle.kind, op, spec, scene.frame, pairs, samples, weighting=scene.weighting,
                        batch_frames=batch_frames, keep_maps=maps != "none")
    write_map_csv(out_path, scene.grid, res, truth, map_rows=maps == "csv")
    if maps == "npy":
        np.save(out_path.rsplit(".", 1)[0] + "_maps.npy", res.maps)
    return res


def main(argv=None) -> int:
    import argparse
    ap = argparse.ArgumentParser(prog="python -m paper_2306_08514_b200.batch",
                                 description="Batched GPU `map` over a recording (reference cli.py:210-259).")
    sub = ap.add_subparsers(dest="cmd", required=True)
    pm = sub.add_parser("map")
    pm.add_argument("--config", required=True)
    pm.add_argument("--cache", required=True)
    pm.add_argument("--audio", required=True)
    pm.add_argument("--out", required=True)
    pm.add_argument("--truth")
    pm.add_argument("--maps", default="none", choices=["none", "csv", "npy"])
    pm.add_argument("--batch-frames", type=int, default=4096)
    a = ap.parse_args(argv)
    cmd_map(read_run_config(a.config), a.cache, a.audio, a.out, a.truth, maps=a.maps,
            batch_frames=a.batch_frames)
    print(f"map CSV written to {a.out}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
