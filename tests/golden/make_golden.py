"""Generate golden vectors by importing the reference `srpmap` package itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes small .npz fixtures next to this script.  They pin both the CPU oracle
(`oracle/srp_oracle.py`) and the GPU path.  Nothing at test/bench time reads
/root/reference; only these committed fixtures travel to the GPU box.

The scenes mirror the reference test fixtures' shapes (tests/conftest.py:52-97)
plus a reduced BASELINE cfg1 scene; inputs are seeded synthetic arrays.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import srpmap  # noqa: E402
from srpmap import (FdGcc, FrameSpec, MicrophoneArray, SampleSpec, TdoaTable,  # noqa: E402
                    build_ff_grid, build_interp_matrix, build_nf_grid,
                    build_srp_matrix, enumerate_pairs, fd_gcc, locate, lr_map,
                    sample_spec, si_map, slri_map, srp_map_exact, sspi_map,
                    stft_frame, td_gcc_samples, tdoa_table, truncate_low_rank,
                    truncate_sparse, truncate_srp_matrix)
from srpmap.frontend import frame_window  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def _save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def scene_case(name, mode, positions, c, grid, frame, n_aux, keeps, ranks, frames, seed,
               hann=False, signal_len=None, extra_sp=None):
    array = MicrophoneArray(np.asarray(positions, float), c)
    pairs = enumerate_pairs(array)
    tdoa = tdoa_table(array, pairs, grid)
    spec = sample_spec(tdoa, frame, n_aux)
    rng = np.random.default_rng(seed)
    m = array.num_mics
    n = signal_len or (frames - 1) * frame.hop + frame.frame_len
    samples = 0.3 * rng.standard_normal((m, n))
    # a common source with per-channel integer delays so the maps have a peak
    common = rng.standard_normal(n + 16)
    delays = rng.integers(0, 4, m)
    for ch in range(m):
        samples[ch] += common[delays[ch]:delays[ch] + n]
    win = frame_window(frame)
    if hann:
        win = 0.5 - 0.5 * np.cos(2 * np.pi * np.arange(frame.frame_len) / frame.frame_len)
    spectra = []
    for f in range(frames):
        if hann:
            seg = samples[:, f * frame.hop:f * frame.hop + frame.frame_len]
            spectra.append(np.fft.rfft(seg * win[None, :], axis=1))
        else:
            spectra.append(stft_frame(samples, frame, f))
    spectra = np.stack(spectra)
    gccs = [fd_gcc(s, pairs) for s in spectra]
    psi = np.stack([g.values for g in gccs])
    psi_none = np.stack([fd_gcc(s, pairs, weighting="none").values for s in spectra])
    xi_ifft = np.stack([td_gcc_samples(g, spec, "ifft").values for g in gccs])
    xi_matrix = np.stack([td_gcc_samples(g, spec, "matrix").values for g in gccs])
    srp = build_srp_matrix(tdoa, frame, max_bytes=1 << 34)
    z_conv = np.stack([srp_map_exact(srp, g) for g in gccs])
    interp = build_interp_matrix(tdoa, spec, frame, max_bytes=1 << 34)
    z_si = np.stack([si_map(interp, x) for x in xi_ifft])
    out = dict(positions=array.positions, speed_of_sound=np.float64(c),
               grid_points=grid.points, grid_mode=np.array(grid.mode),
               frame_len=np.int64(frame.frame_len), sample_rate=np.float64(frame.sample_rate),
               hop=np.int64(frame.hop), window=win, hann=np.bool_(hann), n_aux=np.int64(n_aux),
               pairs=pairs.pairs, distances=pairs.distances,
               delta_t=tdoa.delta_t, limits=tdoa.limits, counts=spec.counts,
               offsets=spec.offsets, samples=samples, spectra=spectra, psi=psi,
               psi_none=psi_none, xi_ifft=xi_ifft, xi_matrix=xi_matrix,
               z_conv=z_conv, interp=interp.matrix, z_si=z_si,
               argmax_conv=np.array([locate(z, grid)[0] for z in z_conv]))
    jp = grid.num_points * pairs.num_pairs
    for q in keeps:
        keep = interp.matrix.size if q == "all" else int(round(q * jp))
        sp = truncate_sparse(interp, keep)
        tag = "all" if q == "all" else f"{q}jp".replace(".", "p")
        if q != "all":  # keep-all structure is the full dense pattern
            out[f"sp_{tag}_values"] = sp.values
            out[f"sp_{tag}_cols"] = sp.col_indices.astype(np.int32)
            out[f"sp_{tag}_splits"] = sp.row_splits
        out[f"sp_{tag}_keep"] = np.int64(keep)
        out[f"z_sspi_{tag}"] = np.stack([sspi_map(sp, x) for x in xi_ifft])
    for r in ranks:
        lr = truncate_low_rank(interp, r)
        out[f"slri_{r}_tall"] = lr.tall
        out[f"slri_{r}_fat"] = lr.fat
        out[f"z_slri_{r}"] = np.stack([slri_map(lr, x) for x in xi_ifft])
        lrs = truncate_srp_matrix(srp, r)
        out[f"lr_{r}_tall"] = lrs.tall
        out[f"lr_{r}_fat"] = lrs.fat
        out[f"z_lr_{r}"] = np.stack([lr_map(lrs, g) for g in gccs])
    out["keeps"] = np.array([str(q) for q in keeps])
    out["ranks"] = np.array(ranks, dtype=np.int64)
    _save(name, **out)


def known_answers():
    """Known-answer vectors from the reference tests (cited file:line)."""
    out = {}
    # test_srp.py:27-32: K=2, dt=T -> H entry j
    frame = FrameSpec(frame_len=4, sample_rate=100)
    srp = build_srp_matrix(TdoaTable(np.array([[0.01]]), np.array([1.01])), frame)
    out["ka_h_entry"] = srp.matrix
    # test_srp.py:56-65: single active bin -> 2 cos(w_k dt)
    frame = FrameSpec(frame_len=8, sample_rate=800)
    dt = np.array([[0.0], [0.5e-3], [1.0e-3]])
    srp = build_srp_matrix(TdoaTable(dt, np.array([2.0e-3])), frame)
    vals = np.zeros(3, complex)
    vals[0] = 1.0
    out["ka_cos_dt"] = dt
    out["ka_cos_z"] = srp_map_exact(srp, FdGcc(vals, 1, 3, "none"))
    # test_sampling.py:67-79: single bin -> sampled cosine (three-pair spec)
    frame = FrameSpec(frame_len=32, sample_rate=1000)
    t = frame.sample_period
    tdoa = TdoaTable(np.zeros((1, 3)), np.array([2.2 * t, 3.4 * t, 4.1 * t]))
    spec = sample_spec(tdoa, frame, n_aux=0)
    per = np.zeros((3, frame.num_bins), complex)
    per[:, 4] = 1.0
    g = FdGcc(per.ravel(), 3, frame.num_bins, "none")
    out["ka_cos_counts"] = spec.counts
    out["ka_cos_xi"] = td_gcc_samples(g, spec, "ifft").values
    # test_sampling.py:51-55 lag layout; :22-27 N_p = 77
    frame = FrameSpec(frame_len=64, sample_rate=8000)
    spec = sample_spec(TdoaTable(np.zeros((1, 1)), np.array([2.4e-4])), frame, n_aux=1)
    out["ka_lag_layout"] = spec.lag_indices(0)
    spec = sample_spec(TdoaTable(np.zeros((1, 1)), np.array([6.4 / 340.0])),
                       FrameSpec(frame_len=512, sample_rate=4000), n_aux=2)
    out["ka_count_77"] = spec.counts
    # test_sampling.py:29-35: hexagonal ring, 30 deg FF grid -> S = 699
    array = MicrophoneArray.circular((0, 0, 0), 0.3, 6)
    tdoa = tdoa_table(array, enumerate_pairs(array), build_ff_grid(30.0))
    out["ka_hex_total"] = np.int64(sample_spec(tdoa, FrameSpec(1024, 16000)).total_samples)
    # test_interpolation.py:157-163: top-Q selection and row-major tie-break
    spec0 = SampleSpec(np.zeros(3, np.int64), 0, 64)
    sp = truncate_sparse(srpmap.InterpMatrix(np.array([[0.9, -0.5, 0.1], [0.2, -0.8, 0.3]]),
                                             spec0), 2)
    out["ka_topq_dense"] = sp.to_dense()
    spec0 = SampleSpec(np.zeros(2, np.int64), 0, 64)
    sp = truncate_sparse(srpmap.InterpMatrix(np.array([[0.5, -0.5], [0.5, 0.5]]), spec0), 2)
    out["ka_tie_dense"] = sp.to_dense()
    # test_frontend.py:89-100: integer circular delay -> exact phase ramp (rect window)
    spec = FrameSpec(frame_len=32, sample_rate=1000, window="rect")
    x = np.random.default_rng(4).standard_normal(32)
    sig = np.stack([np.roll(x, 3), x])
    pairs = enumerate_pairs(MicrophoneArray(np.array([[0.0, 0, 0], [0.1, 0, 0]])))
    out["ka_ramp_signal"] = sig
    out["ka_ramp_psi"] = fd_gcc(stft_frame(sig, spec, 0), pairs).values
    # test_frontend.py:137-145: floored bin is exactly 0
    rng = np.random.default_rng(8)
    spectra = rng.standard_normal((2, 33)) + 1j * rng.standard_normal((2, 33))
    spectra[1, 5] = 0.0
    out["ka_floor_spectra"] = spectra
    out["ka_floor_psi"] = fd_gcc(spectra, pairs).values
    # test_srp.py:101-105: argmax tie -> lower index
    out["ka_tie_z"] = np.array([0.0, 5.0, 5.0, 1.0])
    out["ka_tie_index"] = np.int64(np.argmax(out["ka_tie_z"]))
    _save("known_answers", **out)


def main():
    known_answers()
    # reference conftest nf_mini-like scene (tests/conftest.py:52-57), 4 kHz, K=256
    nf_pos = np.array([[0.45, 0.45, 1.0], [4.45, 0.45, 3.0], [0.45, 5.45, 3.0],
                       [4.45, 5.45, 1.0]])
    scene_case("nf_mini", "nf", nf_pos, 340.0,
               build_nf_grid((2.15, 2.65, 1.45), (0.6, 0.6, 0.1), 0.1),
               FrameSpec(frame_len=512, sample_rate=4000), 2,
               keeps=[0, 1, 2, 4, "all"], ranks=[1, 4], frames=6, seed=101)
    # reference conftest ff_mini-like scene (tests/conftest.py:60-65), ring r=0.3
    ring = MicrophoneArray.circular((3.25, 4.5, 1.0), 0.3, 6)
    scene_case("ff_mini", "ff", ring.positions, 340.0, build_ff_grid(15.0),
               FrameSpec(frame_len=1024, sample_rate=16000), 2,
               keeps=[0.5, 1, 2, 3, "all"], ranks=[2, 8], frames=5, seed=102)
    # BASELINE cfg1 geometry (M=4 in a 0.5 m square, c=343, 16 kHz, K=512, Hann),
    # grid reduced to 0.4 m to keep the fixture small
    rng = np.random.default_rng(7)
    pos = np.column_stack([rng.uniform(1.75, 2.25, 4), rng.uniform(1.75, 2.25, 4), np.zeros(4)])
    scene_case("cfg1_small", "nf", pos, 343.0,
               build_nf_grid((0, 0, 0), (4, 4, 0), 0.4),
               FrameSpec(frame_len=1024, sample_rate=16000), 2,
               keeps=[1, 2, "all"], ranks=[4], frames=4, seed=103, hann=True)
    # BASELINE cfg3 geometry (UCA M=8 r=5 cm, c=343, K=256, Hann), 10 deg grid
    uca = MicrophoneArray.circular((0, 0, 0), 0.05, 8, 343.0)
    scene_case("cfg3_small", "ff", uca.positions, 343.0, build_ff_grid(10.0),
               FrameSpec(frame_len=512, sample_rate=16000), 2,
               keeps=[1, 2, "all"], ranks=[4], frames=4, seed=104, hann=True)


if __name__ == "__main__":
    main()
