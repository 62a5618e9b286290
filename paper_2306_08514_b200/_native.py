"""ctypes binding of the C-ABI in include/srpgpu.h (libsrpgpu.so, built in-tree).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every op raises `NativeLibraryError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import CapacityError, DimensionError, NativeLibraryError

LIB_PATH = os.environ.get("SRPGPU_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                        "libsrpgpu.so")

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_F32 = ctypes.c_float
_F64 = ctypes.c_double

# name -> argtypes (restype is int status unless listed in _RESTYPES)
SIGNATURES = {
    "srpgpu_last_error": [],
    "srpgpu_abi_version": [],
    "srpgpu_launch_count": [],
    "srpgpu_device_sync": [],
    "srpgpu_set_frontend_kernel": [_I32],
    "srpgpu_stft": [_P, _I32, _I64, _I64, _P, _I32, _I32, _I64, _I64, _P, _P, _P],
    "srpgpu_fd_gcc": [_P, _I64, _I32, _I32, _P, _I32, _I32, _I32, _F64, _P, _P],
    "srpgpu_gcc_frames": [_P, _I32, _I64, _I64, _P, _I32, _I32, _I64, _I64, _P, _I32, _I32, _I32,
                          _F64, _P, _I64, _I32, _P],
    "srpgpu_td_gcc_samples": [_P, _I64, _I32, _I32, _P, _P, _I32, _P, _I64, _P],
    "srpgpu_frames_to_samples": [_P, _I32, _I64, _I64, _P, _I32, _I32, _I64, _I64, _P, _I32, _I32,
                                 _I32, _F64, _P, _P, _I32, _P, _I64, _P],
    "srpgpu_frames_to_samples_planes": [_P, _I32, _I64, _I64, _P, _I32, _I32, _I64, _I64, _P, _I32,
                                        _I32, _I32, _F64, _P, _P, _I32, _P, _I64, _P, _I32, _I64, _I32, _P, _P],
    "srpgpu_frames_to_sspi_map": [_P, _I32, _I64, _I64, _P, _I32, _I32, _I64, _I64, _P, _I32, _I32, _I32,
                                  _F64, _P, _P, _I32, _P, _P, _P, _I64, _P, _P, _P, _P],
    "srpgpu_frames_to_slri_map": [_P, _I32, _I64, _I64, _P, _I32, _I32, _I64, _I64, _P, _I32, _I32, _I32,
                                  _F64, _P, _P, _I32, _P, _P, _I32, _I64, _P, _P, _P, _P],
    "srpgpu_spectra_to_samples": [_P, _I64, _I32, _I32, _P, _I32, _I32, _I32, _F64, _P, _P, _I32,
                                  _P, _I64, _P],
    "srpgpu_render_images": [_P, _I64, _I32, _I32, _P, _P, _P, _P, _P, _P, _P],
    "srpgpu_sspi_map": [_P, _I64, _I64, _I32, _I32, _P, _P, _I64, _I64, _I64, _P, _P, _P],
    "srpgpu_transpose": [_P, _I64, _I64, _I64, _P, _I64, _P],
    "srpgpu_interp_map_tc": [_P, _I64, _P, _I64, _I32, _P, _P, _P],
    "srpgpu_split_bf16": [_P, _I64, _I32, _I64, _I32, _P, _I32, _P],
    "srpgpu_split_bf16_cols": [_P, _I64, _I32, _I64, _I32, _P, _P, _I32, _P],
    "srpgpu_interp_map_gather_tc": [_P, _I64, _I32, _I64, _P, _I64, _P, _P, _P, _P, _I32, _I64, _I32, _P, _P,
                                    _P, _P, _P],
    "srpgpu_interp_map_gather_tf32": [_P, _I64, _I32, _I64, _P, _I64, _P, _P, _P, _P, _I32, _I64, _I32, _P, _P,
                                      _P, _P, _P],
    "srpgpu_interp_map_gather_f16": [_P, _I64, _I32, _I64, _P, _I64, _P, _P, _P, _P, _I32, _I64, _I32, _P, _F32,
                                     _P, _P, _P, _P],
    "srpgpu_interp_map_untile": [_P, _I32, _P, _I64, _I64, _P, _I32, _P],
    "srpgpu_split_f16_rows": [_P, _I64, _I64, _I64, _P, _F32, _P, _I64, _I64, _P],
    "srpgpu_split_bf16_rows": [_P, _I64, _I64, _I64, _P, _P, _I64, _I64, _P],
    "srpgpu_split_tf32_rows": [_P, _I64, _I64, _I64, _P, _P, _I64, _I64, _P],
    "srpgpu_slri_map": [_P, _I64, _I64, _I32, _P, _P, _I32, _I64, _P, _P, _P, _P],
    "srpgpu_slri_map_tc": [_P, _I64, _I64, _I32, _P, _P, _I32, _I32, _I64, _P, _P, _P, _P, _P],
    "srpgpu_lr_map_tc": [_P, _I64, _I32, _P, _P, _I32, _I32, _I64, _P, _P, _P, _P, _P],
    "srpgpu_lr_map": [_P, _I64, _I32, _P, _P, _I32, _I64, _P, _P, _P, _P],
    "srpgpu_srp_map_simt": [_P, _I64, _I32, _P, _I64, _P, _P, _P],
    "srpgpu_srp_map_tc": [_P, _I64, _I64, _I32, _P, _I64, _I64, _I32, _P, _P, _P, _P],
    "srpgpu_srp_map_tdoa": [_P, _I64, _I64, _I32, _I32, _P, _I64, _I32, _I32, _P, _P, _P, _P],
    "srpgpu_split_tf32": [_P, _I64, _P, _I64, _I64, _I64, _P],
    "srpgpu_round_tf32": [_P, _I64, _P, _I64, _I64, _I64, _P],
    "srpgpu_c128_to_steering": [_P, _I64, _I64, _I64, _P, _I64, _I32, _P],
    "srpgpu_gemm_nt": [_P, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _F32, _P, _P],
    "srpgpu_argmax": [_P, _I64, _I64, _I64, _P, _P],
    "srpgpu_decode_keys": [_P, _I64, _P, _P, _P],
}
_RESTYPES = {
    "srpgpu_last_error": ctypes.c_char_p,
    "srpgpu_launch_count": ctypes.c_uint64,
}

_lock = threading.Lock()
_lib = None


def load():
    """Load libsrpgpu.so (no GPU needed just to load and inspect symbols)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (nvcc, sm_100a); there is no CPU fallback")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().srpgpu_last_error()
    return msg.decode() if msg else ""


def launch_count() -> int:
    return int(load().srpgpu_launch_count())


def call(name: str, *args) -> None:
    """Invoke a C-ABI entry point; map its status onto the reference's exceptions."""
    status = getattr(load(), name)(*args)
    if status == 0:
        return
    msg = last_error()
    if status == -1:
        raise DimensionError(msg)
    if status in (-2, -5):
        raise ValueError(msg)
    if status == -3:
        raise CapacityError(msg)
    raise NativeLibraryError(f"{name}: {msg} (status {status})")
