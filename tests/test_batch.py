"""Batched `map` command against the reference CLI's own outputs.

Fixtures (tests/golden/cli/, cli_golden.npz) come from the reference itself
(tests/golden/make_cli_golden.py): an INI run configuration, float32 and int16 WAV
recordings, `cmd_precompute` caches (sspi, conv) and `cmd_map` CSVs with a truth.
"""

import csv
import os

import numpy as np
import pytest

import paper_2306_08514_b200 as s
from paper_2306_08514_b200 import batch as B

HERE = os.path.dirname(os.path.abspath(__file__))
CLI = os.path.join(HERE, "golden", "cli")
TRUTH = "0.5 0.5 0"


def read_rows(path):
    with open(path, newline="") as fh:
        rows = list(csv.reader(fh))
    assert rows[0] == B.CSV_HEADER
    maps = [r for r in rows[1:] if r[0] == "map"]
    summ = [r for r in rows[1:] if r[0] == "summary"]
    return maps, summ


@pytest.fixture(scope="module")
def golden():
    return dict(np.load(os.path.join(HERE, "golden", "cli_golden.npz")))


@pytest.mark.parametrize("tag", ["f32", "i16"])
def test_load_audio_matches_reference(golden, tag):
    x, rate = B.load_audio(os.path.join(CLI, f"scene_{tag}.wav"))
    assert x.dtype == np.float32 and rate == float(golden[f"rate_{tag}"])
    assert np.array_equal(x.astype(np.float64), golden[f"audio_{tag}"])     # exact: both formats fit f32


def test_load_audio_raw(tmp_path):
    x = np.arange(12, dtype="<f4")
    p = tmp_path / "a.f32"
    x.tofile(p)
    y, rate = B.load_audio(str(p), sample_rate=8000, channels=3)
    assert rate == 8000.0 and np.array_equal(y, x.reshape(-1, 3).T)
    with pytest.raises(ValueError):
        B.load_audio(str(p))
    with pytest.raises(ValueError):
        B.load_audio(str(p), sample_rate=8000, channels=5)


@pytest.mark.parametrize("kind", ["sspi", "conv"])
def test_run_config_reproduces_cache_digest(kind):
    scene = B.read_run_config(os.path.join(CLI, "run.ini"))
    b = s.load_cache(os.path.join(CLI, f"{kind}.srpm"))
    assert B.scene_hash(scene, b.kind, b.meta) == b.params_hash
    other = B.RunScene(scene.mode, scene.room, scene.array, scene.grid, scene.frame, "none", scene.n_aux)
    assert B.scene_hash(other, b.kind, b.meta) != b.params_hash


def test_csv_rows_format_like_reference():
    """Fed the reference's own maxima and maps, the writer reproduces its CSV byte for byte."""
    scene = B.read_run_config(os.path.join(CLI, "run.ini"))
    ref = os.path.join(CLI, "map_sspi_f32.csv")
    maps, summ = read_rows(ref)
    nf = len(summ)
    j = scene.grid.num_points
    z = np.array([float(r[6]) for r in maps]).reshape(nf, j)
    res = B.RecordingMaps(index=np.array([int(r[2]) for r in summ]),
                          value=np.array([float(r[6]) for r in summ]), maps=z)
    out = "/tmp/_rows.csv"
    B.write_map_csv(out, scene.grid, res, B.parse_truth(TRUTH, scene), map_rows=True)
    assert open(out).read() == open(ref).read()


def test_cmd_map_errors(tmp_path):
    scene = B.read_run_config(os.path.join(CLI, "run.ini"))
    wav = os.path.join(CLI, "scene_f32.wav")
    bad = B.RunScene(scene.mode, scene.room, scene.array, scene.grid, scene.frame, "none", scene.n_aux)
    with pytest.raises(s.ConfigError, match="cache/config mismatch"):
        B.cmd_map(bad, os.path.join(CLI, "sspi.srpm"), wav, str(tmp_path / "o.csv"))
    fr = s.FrameSpec(frame_len=256, sample_rate=8000.0)
    other_rate = B.RunScene(scene.mode, scene.room, scene.array, scene.grid, fr, scene.weighting, scene.n_aux)
    b = s.load_cache(os.path.join(CLI, "sspi.srpm"))
    p2 = str(tmp_path / "c.srpm")
    s.save_cache(p2, b.kind, b.arrays, b.meta, B.scene_hash(other_rate, b.kind, b.meta))
    with pytest.raises(s.ConfigError, match="audio rate"):
        B.cmd_map(other_rate, p2, wav, str(tmp_path / "o.csv"))
    with pytest.raises(s.ConfigError):
        B.parse_truth("1 2", scene)
    with pytest.raises(ValueError):
        B.cmd_map(scene, os.path.join(CLI, "sspi.srpm"), wav, str(tmp_path / "o.csv"), maps="xml")
    with pytest.raises(s.ConfigError):
        B.read_run_config(str(tmp_path / "missing.ini"))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["sspi", "conv"])
@pytest.mark.parametrize("tag", ["f32", "i16"])
def test_gpu_cmd_map_matches_reference(tmp_path, kind, tag):
    scene = B.read_run_config(os.path.join(CLI, "run.ini"))
    ref_maps, ref_summ = read_rows(os.path.join(CLI, f"map_{kind}_{tag}.csv"))
    out = str(tmp_path / "o.csv")
    res = B.cmd_map(scene, os.path.join(CLI, f"{kind}.srpm"), os.path.join(CLI, f"scene_{tag}.wav"), out,
                    TRUTH, maps="csv", batch_frames=5)          # 12 frames: 3 batches, a padded last one
    maps, summ = read_rows(out)
    assert len(summ) == len(ref_summ) == 12 and len(maps) == len(ref_maps)
    j = scene.grid.num_points
    zr = np.array([float(r[6]) for r in ref_maps]).reshape(-1, j)
    zg = np.array([float(r[6]) for r in maps]).reshape(-1, j)
    err = np.abs(zg - zr).max(axis=1) / np.abs(zr).max(axis=1)
    assert err.max() <= 1e-4, f"{kind}/{tag}: {err.max():.2e}"
    srt = np.sort(zr, axis=1)
    margin = (srt[:, -1] - srt[:, -2]) / np.abs(zr).max(axis=1)
    for f, (a, r) in enumerate(zip(summ, ref_summ)):
        assert a[1] == r[1]
        if margin[f] > 1e-4:
            assert a[2:6] == r[2:6] and a[7:] == r[7:]      # index, location, loc_error, accuracy
        assert abs(float(a[6]) - float(r[6])) <= 1e-4 * np.abs(zr[f]).max()
    assert np.array_equal(res.index, [int(r[2]) for r in summ])


@pytest.mark.gpu
def test_gpu_map_recording_batches_agree(tmp_path):
    """Batch size does not change the result (padded tail frames are dropped)."""
    scene = B.read_run_config(os.path.join(CLI, "run.ini"))
    kind, op, spec = s.load_operator(os.path.join(CLI, "sspi.srpm"))
    x, _ = B.load_audio(os.path.join(CLI, "scene_f32.wav"))
    pairs = s.enumerate_pairs(scene.array)
    a = B.map_recording(kind, op, spec, scene.frame, pairs, x, batch_frames=12, keep_maps=True)
    b = B.map_recording(kind, op, spec, scene.frame, pairs, x, batch_frames=7, keep_maps=True)
    assert np.array_equal(a.index, b.index) and np.array_equal(a.maps, b.maps)
    empty = B.map_recording(kind, op, spec, scene.frame, pairs, x[:, :100])
    assert empty.index.shape == (0,)
    B.cmd_map(scene, os.path.join(CLI, "sspi.srpm"), os.path.join(CLI, "scene_f32.wav"),
              str(tmp_path / "o.csv"), maps="npy")
    assert np.load(str(tmp_path / "o_maps.npy")).shape == (12, scene.grid.num_points)
