"""The C-ABI library loads without a GPU and exports every symbol include/srpgpu.h declares."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "srpgpu.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(srpgpu_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2306_08514_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return _native.load()


def test_header_declares_the_path():
    syms = declared_symbols()
    for name in ("srpgpu_stft", "srpgpu_fd_gcc", "srpgpu_td_gcc_samples", "srpgpu_sspi_map",
                 "srpgpu_slri_map", "srpgpu_lr_map", "srpgpu_srp_map_tc", "srpgpu_argmax"):
        assert name in syms


def test_every_declared_symbol_is_exported(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_python_binding_covers_header(lib):
    from paper_2306_08514_b200 import _native
    assert sorted(_native.SIGNATURES) == declared_symbols()


def test_abi_version_and_counter(lib):
    assert lib.srpgpu_abi_version() == 1
    assert isinstance(lib.srpgpu_launch_count(), int)


def test_argument_errors_do_not_touch_the_device(lib):
    # shape validation happens before any CUDA call and maps onto the reference errors
    from paper_2306_08514_b200 import _native
    with pytest.raises(ValueError):
        _native.call("srpgpu_stft", None, 2, 100, 100, None, 12, 6, 0, 1, None, None, None)
    assert "power of two" in _native.last_error()
    with pytest.raises(ValueError):
        _native.call("srpgpu_slri_map", None, 0, 1, 4, None, None, 0, 4, None, None, None, None)
