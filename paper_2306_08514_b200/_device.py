"""Device plumbing: tensor conversion, streams, and the upload-once operator cache.

PyTorch is used only for device memory and streams; all arithmetic on the
per-frame path runs in the sm_100a kernels of libsrpgpu.so.
"""

from __future__ import annotations

import threading
import weakref

import numpy as np
import torch

from .errors import NativeLibraryError


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device: the SRP-map ops run only on the GPU "
                                 "(there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def num_sms() -> int:
    """SM count of the current device (148 on B200)."""
    return torch.cuda.get_device_properties(device()).multi_processor_count


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def as_f32(x, contiguous: bool = True) -> torch.Tensor:
    """Real input on the device as float32 (H2D copy if it came from the host)."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=device(), dtype=torch.float32)
    else:
        arr = np.asarray(x)
        if np.iscomplexobj(arr):
            raise TypeError("expected a real array")
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to(device(), non_blocking=False)
    return t.contiguous() if contiguous else t


def as_c64(x) -> torch.Tensor:
    """Complex input on the device as complex64, contiguous."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=device())
        if not t.is_complex():
            t = t.to(torch.complex64)
        return t.to(torch.complex64).contiguous()
    arr = np.ascontiguousarray(np.asarray(x), dtype=np.complex64)
    return torch.from_numpy(arr).to(device())


def as_i32(x) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x), dtype=np.int32)).to(device())


def as_i64(x) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x), dtype=np.int64)).to(device())


class OperatorCache:
    """Device copies of host operators, built once per (operator object, variant).

    Keyed by id() with a weakref finalizer, because the reference's frozen
    dataclasses hold numpy arrays and are not hashable.
    """

    def __init__(self):
        # re-entrant, and no cached value is released while it is held: releasing one can
        # run another entry's weakref finalizer (_drop) on this thread
        self._lock = threading.RLock()
        self._entries: dict = {}

    def get(self, obj, variant, builder):
        key = (id(obj), variant)
        with self._lock:
            hit = self._entries.get(key)
            if hit is not None and hit[0]() is obj:
                return hit[1]
        value = builder()
        try:
            ref = weakref.ref(obj, lambda _r, k=key: self._drop(k))
        except TypeError:  # not weak-referenceable: keep a strong ref
            ref = (lambda o=obj: o)
        with self._lock:
            old = self._entries.get(key)
            self._entries[key] = (ref, value)
        del old                                  # released outside the lock
        return value

    def _drop(self, key):
        with self._lock:
            old = self._entries.pop(key, None)
        del old

    def clear(self):
        with self._lock:
            old = self._entries
            self._entries = {}
        del old


CACHE = OperatorCache()
