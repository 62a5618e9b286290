"""Pin the CPU oracle (oracle/srp_oracle.py) to reference-generated golden vectors.

The fixtures were produced by importing the reference package itself
(tests/golden/make_golden.py); these tests make the oracle trustworthy as the
checker for the GPU path.
"""

import numpy as np
import pytest
from numpy.testing import assert_allclose, assert_array_equal

from oracle import srp_oracle as O
from conftest import keep_tags


def test_geometry_and_counts(golden_scene):
    _, g = golden_scene
    assert_array_equal(O.enumerate_pairs(g["positions"].shape[0]), g["pairs"])
    delta, limits = O.tdoa_table(g["positions"], float(g["speed_of_sound"]), str(g["grid_mode"]),
                                 g["grid_points"])
    assert_array_equal(delta, g["delta_t"])          # same float64 expressions -> bit-exact
    assert_array_equal(limits, g["limits"])
    counts = O.sample_counts(limits, float(g["sample_rate"]), int(g["frame_len"]), int(g["n_aux"]))
    assert_array_equal(counts, g["counts"])
    assert_array_equal(O.sample_offsets(counts), g["offsets"])


def test_frontend(golden_scene):
    _, g = golden_scene
    frames = np.arange(g["spectra"].shape[0])
    spectra = O.stft_frames(g["samples"], int(g["frame_len"]), int(g["hop"]), g["window"], frames)
    assert_allclose(spectra, g["spectra"], rtol=0, atol=1e-10)
    assert_allclose(O.fd_gcc(g["spectra"], g["pairs"]), g["psi"], atol=1e-12)
    assert_allclose(O.fd_gcc(g["spectra"], g["pairs"], "none"), g["psi_none"], rtol=1e-12, atol=1e-9)


def test_sampling_paths(golden_scene):
    _, g = golden_scene
    k = int(g["frame_len"]) // 2
    xi = O.td_gcc_samples(g["psi"], g["counts"], k, "ifft")
    assert_allclose(xi, g["xi_ifft"], rtol=0, atol=1e-9)
    xm = O.td_gcc_samples(g["psi"], g["counts"], k, "matrix")
    assert_allclose(xm, g["xi_matrix"], rtol=0, atol=1e-9)
    assert np.linalg.norm(xi - xm) / np.linalg.norm(xm) < 1e-12


def test_maps(golden_scene):
    _, g = golden_scene
    H = O.build_srp_matrix(g["delta_t"], int(g["frame_len"]), float(g["sample_rate"]))
    z = O.srp_map_exact(H, g["psi"])
    assert_allclose(z, g["z_conv"], rtol=1e-12, atol=1e-9)
    assert_array_equal(O.locate(z), g["argmax_conv"])
    lam = O.build_interp_matrix(g["delta_t"], g["counts"], float(g["sample_rate"]))
    assert_array_equal(lam, g["interp"])
    assert_allclose(O.si_map(lam, g["xi_ifft"]), g["z_si"], rtol=1e-12, atol=1e-9)
    for r in g["ranks"]:
        assert_allclose(O.slri_map(g[f"slri_{r}_tall"], g[f"slri_{r}_fat"], g["xi_ifft"]),
                        g[f"z_slri_{r}"], rtol=1e-10, atol=1e-8)
        assert_allclose(O.lr_map(g[f"lr_{r}_tall"], g[f"lr_{r}_fat"], g["psi"]), g[f"z_lr_{r}"],
                        rtol=1e-10, atol=1e-8)


def test_sparse_fit_bit_exact(golden_scene):
    _, g = golden_scene
    lam = g["interp"]
    for tag in keep_tags(g):
        keep = int(g[f"sp_{tag}_keep"])
        vals, cols, splits = O.truncate_sparse(lam, keep)
        if tag != "all":
            assert_array_equal(vals, g[f"sp_{tag}_values"])
            assert_array_equal(cols, g[f"sp_{tag}_cols"])
            assert_array_equal(splits, g[f"sp_{tag}_splits"])
        assert_allclose(O.sspi_map(vals, cols, splits, g["xi_ifft"]), g[f"z_sspi_{tag}"],
                        rtol=1e-12, atol=1e-9)


def test_known_answers(known):
    H = O.build_srp_matrix(np.array([[0.01]]), 4, 100.0)
    assert_allclose(H, known["ka_h_entry"], atol=1e-15)
    H = O.build_srp_matrix(known["ka_cos_dt"], 8, 800.0)
    v = np.zeros(3, complex)
    v[0] = 1.0
    assert_allclose(O.srp_map_exact(H, v), known["ka_cos_z"], atol=1e-14)
    per = np.zeros((3, 15), complex)
    per[:, 4] = 1.0
    assert_allclose(O.td_gcc_samples(per.ravel(), known["ka_cos_counts"], 16), known["ka_cos_xi"],
                    atol=1e-12)
    assert_array_equal(O.lag_indices(2), known["ka_lag_layout"])
    assert O.sample_counts(np.array([6.4 / 340.0]), 4000.0, 512).tolist() == known["ka_count_77"].tolist()
    vals, cols, splits = O.truncate_sparse(np.array([[0.9, -0.5, 0.1], [0.2, -0.8, 0.3]]), 2)
    dense = np.zeros((2, 3))
    dense[np.repeat(np.arange(2), np.diff(splits)), cols] = vals
    assert_array_equal(dense, known["ka_topq_dense"])
    vals, cols, splits = O.truncate_sparse(np.array([[0.5, -0.5], [0.5, 0.5]]), 2)
    dense = np.zeros((2, 2))
    dense[np.repeat(np.arange(2), np.diff(splits)), cols] = vals
    assert_array_equal(dense, known["ka_tie_dense"])
    win = O.frame_window(32, "rect")
    spectra = O.stft_frames(known["ka_ramp_signal"], 32, 16, win, [0])[0]
    assert_allclose(O.fd_gcc(spectra, np.array([[1, 0]])), known["ka_ramp_psi"], atol=1e-12)
    floor_psi = O.fd_gcc(known["ka_floor_spectra"], np.array([[1, 0]]))
    assert_allclose(floor_psi, known["ka_floor_psi"], atol=1e-15)
    assert floor_psi[4] == 0.0
    assert O.locate(known["ka_tie_z"]) == int(known["ka_tie_index"]) == 1


def test_error_metrics():
    z = np.array([1.0, 2.0, 3.0])
    assert O.map_error(z, z) == -np.inf
    assert O.normalized_max_error(z + 0.03, z)[0] == pytest.approx(0.01)
    assert O.peak_margin(np.array([[0.0, 1.0, 3.0]]))[0] == pytest.approx(2.0 / 3.0)
