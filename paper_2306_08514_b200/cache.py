"""SRPM v1 operator caches straight into device operators.

The reference persists fitted operators in a versioned binary container
(cache.py:1-19 of the reference): magic "SRPM", u16 version 1, u16 reserved, u32
header length, a JSON header (sorted keys: arrays [{name, dtype, shape}], kind,
meta, params_hash), then the raw C-order little-endian payloads (<f8, <c16, <i8).
`cmd_map` (cli.py:210-222) refuses a cache whose params_hash does not match the
run configuration and rebuilds the operator with `operator_from_bundle`
(cli.py:133-159).

This module reads and writes the same files and adds the device side:

* `save_cache` writes byte-identical files to the reference writer;
* `load_cache` memory-maps the payload (a cfg3 "conv" cache is 3.7 GB) and
  raises `CacheFormatError` on the same defects as the reference reader;
* `params_hash` reproduces the reference digest (cli.py:46-66);
* `load_operator` checks the digest, rebuilds the operator and uploads its
  device layout once: the steering matrix is shipped as float64 blocks and
  converted on the GPU (`srpgpu_c128_to_steering`); sparse fits become the
  tiled-band image; low-rank factors are cast once.
"""

from __future__ import annotations

import hashlib
import json
import os
import struct
from dataclasses import dataclass

import numpy as np

from .errors import CacheFormatError, ConfigError

MAGIC = b"SRPM"
VERSION = 1
_PREFIX = struct.Struct("<4sHHI")          # magic, version, reserved, header length
_WIRE = {"<f8": np.dtype("<f8"), "<c16": np.dtype("<c16"), "<i8": np.dtype("<i8")}
KINDS = ("conv", "lr", "si", "slri", "sspi")


@dataclass(frozen=True)
class CacheBundle:
    kind: str
    meta: dict
    arrays: dict
    params_hash: str


def _wire_name(arr: np.ndarray) -> str:
    k = arr.dtype.kind
    if k == "f":
        return "<f8"
    if k == "c":
        return "<c16"
    if k in "iu":
        return "<i8"
    raise CacheFormatError(f"unsupported array dtype {arr.dtype}")


def save_cache(path: str, kind: str, arrays: dict, meta: dict, params_hash: str) -> None:
    """Write an operator bundle (same bytes as the reference writer, cache.py:56-76)."""
    entries, blobs = [], []
    for name, a in arrays.items():
        a = np.asarray(a)
        wire = _wire_name(a)
        entries.append({"name": name, "dtype": wire, "shape": list(a.shape)})
        blobs.append(np.ascontiguousarray(a).astype(_WIRE[wire], copy=False))
    header = json.dumps({"arrays": entries, "kind": kind, "meta": meta, "params_hash": params_hash},
                        sort_keys=True, separators=(",", ":")).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(_PREFIX.pack(MAGIC, VERSION, 0, len(header)))
        fh.write(header)
        for b in blobs:
            fh.write(b.tobytes(order="C"))


def load_cache(path: str, mmap: bool = True) -> CacheBundle:
    """Read a bundle written by `save_cache` or by the reference (cache.py:79-111).

    Payload arrays are read-only memory maps of the file when `mmap` (no copy of a
    multi-GB operator through host RAM), otherwise private copies.
    """
    path = str(path)
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        prefix = fh.read(_PREFIX.size)
        if len(prefix) < 4 or prefix[:4] != MAGIC:
            raise CacheFormatError(f"{path}: not an operator cache (bad magic bytes)")
        if len(prefix) < _PREFIX.size:
            raise CacheFormatError(f"{path}: truncated header")
        _, version, _, hlen = _PREFIX.unpack(prefix)
        if version != VERSION:
            raise CacheFormatError(f"{path}: unsupported cache version {version}")
        start = _PREFIX.size + hlen
        if start > size:
            raise CacheFormatError(f"{path}: truncated header")
        raw = fh.read(hlen)
    try:
        header = json.loads(raw.decode("utf-8"))
        entries = header["arrays"]
    except (UnicodeDecodeError, ValueError, KeyError, TypeError) as exc:
        raise CacheFormatError(f"{path}: corrupt header") from exc
    arrays, off = {}, start
    for e in entries:
        dt = _WIRE.get(e["dtype"])
        if dt is None:
            raise CacheFormatError(f"{path}: unknown dtype {e['dtype']!r}")
        shape = tuple(int(d) for d in e["shape"])
        count = int(np.prod(shape)) if shape else 1
        nbytes = count * dt.itemsize
        if off + nbytes > size:
            raise CacheFormatError(f"{path}: truncated payload for {e['name']!r}")
        if count == 0:
            a = np.zeros(shape, dtype=dt)
        elif mmap:
            a = np.memmap(path, dtype=dt, mode="r", offset=off, shape=shape)
        else:
            a = np.fromfile(path, dtype=dt, count=count, offset=off).reshape(shape)
        arrays[e["name"]] = a
        off += nbytes
    return CacheBundle(kind=header["kind"], meta=header["meta"], arrays=arrays,
                       params_hash=header["params_hash"])


def params_hash(*, mode: str, room, positions, speed_of_sound: float, grid_axes, frame_len: int,
                sample_rate: float, hop: int, weighting: str, n_aux: int, method: str, rank=None,
                keep=None, path: str = "auto") -> str:
    """The digest tying a cache to scene, pipeline and method (cli.py:46-66)."""
    payload = {
        "mode": mode,
        "room": np.asarray(room, dtype=float).tolist(),
        "positions": np.asarray(positions, dtype=float).tolist(),
        "speed_of_sound": float(speed_of_sound),
        "grid_axes": [np.asarray(a).tolist() for a in grid_axes],
        "frame_len": int(frame_len),
        "sample_rate": float(sample_rate),
        "hop": int(hop),
        "weighting": weighting,
        "n_aux": int(n_aux),
        "method": method,
        "rank": rank,
        "keep": keep,
        "path": path,
    }
    text = json.dumps(payload, sort_keys=True, separators=(",", ":"))
    return hashlib.sha256(text.encode("utf-8")).hexdigest()


def operator_from_bundle(bundle: CacheBundle):
    """(operator, SampleSpec or None) rebuilt from a bundle (cli.py:133-159)."""
    from .operators import InterpMatrix, LowRankInterp, LowRankSrp, SparseInterp, SrpMatrix
    from .sampling import SampleSpec
    meta, a, kind = bundle.meta, bundle.arrays, bundle.kind
    if kind not in KINDS:
        raise ConfigError(f"cache holds unknown operator kind {kind!r}")
    if kind == "conv":
        return SrpMatrix(matrix=a["matrix"], num_pairs=meta["num_pairs"], num_bins=meta["num_bins"]), None
    if kind == "lr":
        return LowRankSrp(tall=a["tall"], fat=a["fat"], singular_values=a["singular_values"]), None
    spec = SampleSpec(counts=np.asarray(a["counts"]), n_aux=meta["n_aux"], half_len=meta["half_len"])
    if kind == "si":
        return InterpMatrix(matrix=a["matrix"], spec=spec), spec
    if kind == "slri":
        return LowRankInterp(tall=a["tall"], fat=a["fat"], singular_values=a["singular_values"]), spec
    return SparseInterp(values=a["values"], col_indices=a["col_indices"], row_splits=a["row_splits"],
                        num_cols=meta["num_cols"]), spec


def upload(kind: str, op, spec=None) -> None:
    """Build and cache the operator's device layout now (not on the first map call)."""
    from . import maps
    from .sampling import spec_offsets
    if kind == "conv":
        maps.steering_device(op, tf32=True)
    elif kind == "lr":
        maps._lr_device(op)
    elif kind == "slri":
        maps._slri_device(op)
    elif kind == "sspi":
        maps.band_from_sparse(op, spec_offsets(spec))
    elif kind == "si":
        maps.band_from_dense(op, spec_offsets(spec))
    else:
        raise ConfigError(f"cache holds unknown operator kind {kind!r}")


def load_operator(path: str, expected_hash: str | None = None, *, device: bool = True):
    """(kind, operator, spec) from an SRPM cache, device layout uploaded once.

    `expected_hash` (from `params_hash` of the run configuration) reproduces the
    reference's refusal of a mismatched cache (cli.py:217-222).
    """
    bundle = load_cache(path)
    if expected_hash is not None and bundle.params_hash != expected_hash:
        raise ConfigError("cache/config mismatch: the cache was built for a different "
                          "scene, pipeline, or method; refusing to run")
    op, spec = operator_from_bundle(bundle)
    if device:
        upload(bundle.kind, op, spec)
    return bundle.kind, op, spec
