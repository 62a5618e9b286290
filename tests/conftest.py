"""Shared fixtures.  GPU tests are marked `gpu`; everything else runs on CPU."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
SCENES = ("nf_mini", "ff_mini", "cfg1_small", "cfg3_small")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the sm_100a library")


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session", params=SCENES)
def golden_scene(request):
    return request.param, load_golden(request.param)


@pytest.fixture(scope="session")
def known():
    return load_golden("known_answers")


def scene_objects(g: dict):
    """Product host objects rebuilt from a golden scene's raw parameters."""
    import paper_2306_08514_b200 as s
    array = s.MicrophoneArray(g["positions"], float(g["speed_of_sound"]))
    pairs = s.enumerate_pairs(array)
    grid = s.CandidateGrid(str(g["grid_mode"]), g["grid_points"])
    window = "hann" if bool(g["hann"]) else "sqrt_hann"
    frame = s.FrameSpec(int(g["frame_len"]), float(g["sample_rate"]), int(g["hop"]), window)
    tdoa = s.tdoa_table(array, pairs, grid)
    spec = s.sample_spec(tdoa, frame, int(g["n_aux"]))
    return array, pairs, grid, frame, tdoa, spec


def sparse_from_golden(g: dict, tag: str):
    import paper_2306_08514_b200 as s
    if tag == "all":
        mat = g["interp"]
        j, n = mat.shape
        return s.SparseInterp(mat.ravel().copy(), np.tile(np.arange(n), j).astype(np.int64),
                              np.arange(j + 1, dtype=np.int64) * n, n)
    return s.SparseInterp(g[f"sp_{tag}_values"], g[f"sp_{tag}_cols"].astype(np.int64),
                          g[f"sp_{tag}_splits"], int(g["interp"].shape[1]))


def keep_tags(g: dict):
    out = []
    for q in g["keeps"]:
        q = str(q)
        out.append("all" if q == "all" else (q + "jp").replace(".", "p"))
    return out
