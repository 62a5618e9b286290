"""SRPM operator caches: reference-written files in, device operators out.

Fixtures (tests/golden/cache/*.srpm, cache_golden.npz) were written by the reference
itself (tests/golden/make_cache_golden.py): its builders, `save_cache`, `params_hash`
and the maps `cli.evaluate_map` computes from the operator it reads back.
"""

import os

import numpy as np
import pytest
import torch

import paper_2306_08514_b200 as s
from paper_2306_08514_b200 import cache as C
from oracle import srp_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
CDIR = os.path.join(HERE, "golden", "cache")
KINDS = ("conv", "lr", "si", "slri", "sspi")


@pytest.fixture(scope="module")
def golden():
    return dict(np.load(os.path.join(HERE, "golden", "cache_golden.npz")))


def scene(g):
    array = s.MicrophoneArray(g["positions"], float(g["speed_of_sound"]))
    pairs = s.enumerate_pairs(array)
    frame = s.FrameSpec(frame_len=int(g["frame_len"]), sample_rate=float(g["sample_rate"]))
    return array, pairs, frame


def digest_for(g, kind, meta):
    return C.params_hash(mode="nf", room=g["room"], positions=g["positions"],
                         speed_of_sound=float(g["speed_of_sound"]),
                         grid_axes=[g["grid_axes_x"], g["grid_axes_y"], g["grid_axes_z"]],
                         frame_len=int(g["frame_len"]), sample_rate=float(g["sample_rate"]),
                         hop=int(g["hop"]), weighting="phat", n_aux=int(g["n_aux"]), method=kind,
                         rank=meta.get("rank"), keep=meta.get("keep"), path=meta.get("path", "auto"))


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("mmap", [True, False])
def test_reference_files_round_trip_byte_exact(kind, mmap, tmp_path):
    """Reading a reference-written cache and writing it back reproduces the file byte for byte."""
    src = os.path.join(CDIR, f"{kind}.srpm")
    b = s.load_cache(src, mmap=mmap)
    assert b.kind == kind
    out = tmp_path / "again.srpm"
    s.save_cache(str(out), b.kind, b.arrays, b.meta, b.params_hash)
    assert out.read_bytes() == open(src, "rb").read()


@pytest.mark.parametrize("kind", KINDS)
def test_params_hash_matches_reference_digest(golden, kind):
    b = s.load_cache(os.path.join(CDIR, f"{kind}.srpm"))
    assert b.params_hash == str(golden[f"{kind}_digest"])
    assert digest_for(golden, kind, b.meta) == b.params_hash
    other = dict(b.meta, rank=(b.meta.get("rank") or 0) + 1)
    assert digest_for(golden, kind, other) != b.params_hash


@pytest.mark.parametrize("kind", KINDS)
def test_operator_from_bundle_and_oracle_maps(golden, kind):
    """Rebuilt operators have the reference types/shapes; the oracle maps them to the
    reference's own maps (pins the oracle on cache-loaded operators)."""
    array, pairs, frame = scene(golden)
    b = s.load_cache(os.path.join(CDIR, f"{kind}.srpm"))
    op, spec = s.operator_from_bundle(b)
    x = golden["samples"]
    nf = golden[f"{kind}_z"].shape[0]
    win = O.frame_window(frame.frame_len, frame.window)
    spectra = O.stft_frames(x, frame.frame_len, frame.hop, win, np.arange(nf))
    psi = O.fd_gcc(spectra, pairs.pairs)
    if kind == "conv":
        assert isinstance(op, s.SrpMatrix) and spec is None
        z = O.srp_map_exact(op.matrix, psi)
    elif kind == "lr":
        assert isinstance(op, s.LowRankSrp) and spec is None
        z = O.lr_map(op.tall, op.fat, psi)
    else:
        assert spec is not None and np.array_equal(spec.counts, b.arrays["counts"])
        xi = O.td_gcc_samples(psi, spec.counts, frame.half_len)
        if kind == "si":
            z = xi @ np.asarray(op.matrix).T
        elif kind == "slri":
            z = O.slri_map(op.tall, op.fat, xi)
        else:
            assert isinstance(op, s.SparseInterp) and op.num_cols == b.meta["num_cols"]
            z = O.sspi_map(op.values, op.col_indices, op.row_splits, xi)
    np.testing.assert_allclose(z, golden[f"{kind}_z"], rtol=0, atol=1e-10 * np.abs(golden[f"{kind}_z"]).max())


def test_format_errors(tmp_path):
    p = tmp_path / "op.srpm"
    s.save_cache(str(p), "conv", {"m": np.arange(6.0)}, {}, "00")
    good = p.read_bytes()
    for mutate in (lambda b: b"XXXX" + b[4:],                           # magic
                   lambda b: b[:4] + bytes([7]) + b[5:],                # version
                   lambda b: b[:-8],                                    # truncated payload
                   lambda b: b[:12] + b"\xff" + b[13:],                 # corrupt header
                   lambda b: b[:8] + (10 ** 6).to_bytes(4, "little") + b[12:],   # header past EOF
                   lambda b: b[:3]):                                    # truncated prefix
        p.write_bytes(mutate(good))
        with pytest.raises(s.CacheFormatError):
            s.load_cache(str(p))
    with pytest.raises(s.CacheFormatError):
        s.save_cache(str(tmp_path / "x.srpm"), "conv", {"m": np.array(["a"])}, {}, "00")
    with pytest.raises(ValueError):          # CacheFormatError is a ValueError, as in the reference
        s.load_cache(str(p))


def test_empty_arrays_and_unknown_kind(tmp_path):
    p = tmp_path / "e.srpm"
    s.save_cache(str(p), "sspi", {"values": np.zeros(0), "counts": np.zeros((0, 3), np.int64)}, {}, "00")
    b = s.load_cache(str(p))
    assert b.arrays["values"].shape == (0,) and b.arrays["counts"].shape == (0, 3)
    s.save_cache(str(p), "nope", {"m": np.zeros(2)}, {}, "00")
    with pytest.raises(s.ConfigError):
        s.operator_from_bundle(s.load_cache(str(p)))


def test_load_operator_refuses_mismatched_hash():
    with pytest.raises(s.ConfigError, match="cache/config mismatch"):
        s.load_operator(os.path.join(CDIR, "sspi.srpm"), expected_hash="0" * 64, device=False)
    kind, op, spec = s.load_operator(os.path.join(CDIR, "sspi.srpm"), device=False)
    assert kind == "sspi" and isinstance(op, s.SparseInterp)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", KINDS)
def test_gpu_maps_from_cached_operators(golden, kind):
    """load_operator (digest check + device upload) -> GPU maps == the reference's maps."""
    array, pairs, frame = scene(golden)
    path = os.path.join(CDIR, f"{kind}.srpm")
    b = s.load_cache(path)
    k, op, spec = s.load_operator(path, expected_hash=digest_for(golden, kind, b.meta))
    nf = golden[f"{kind}_z"].shape[0]
    gcc = s.gcc_frames(golden["samples"], frame, pairs, range(nf), tf32=(kind == "conv"))
    z = s.evaluate_map(kind, op, spec, frame, gcc, "ifft")
    z = z.float().cpu().numpy()
    ref = golden[f"{kind}_z"]
    err = O.normalized_max_error(z, ref)
    assert err.max() <= 1e-4, f"{kind}: {err.max():.2e}"


@pytest.mark.gpu
def test_gpu_steering_conversion_bit_exact():
    """float64 payload converted on the GPU == host conj -> complex64 -> TF32 (RNE)."""
    from paper_2306_08514_b200 import maps
    b = s.load_cache(os.path.join(CDIR, "conv.srpm"))     # memory-mapped complex128
    op, _ = s.operator_from_bundle(b)
    for tf32 in (True, False):
        dev = maps.steering_device(op, tf32=tf32).cpu().numpy()
        host = np.conj(np.asarray(op.matrix)).astype(np.complex64).view(np.float32)
        if tf32:
            host = maps._tf32_rne_host(host)
        n = host.shape[1]
        assert np.array_equal(dev[:, :n].view(np.uint32), host.view(np.uint32))
        assert not dev[:, n:].any()
