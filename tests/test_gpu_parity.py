"""GPU parity of every hot-path entry point against the reference's golden vectors.

Tolerances (BASELINE.json north_star): FP32 maps within a normalized max error
of 1e-4 of the reference float64 maps, argmax identical wherever the float64
map's peak margin exceeds 1e-4, sparse structure bit-exact.  Intermediate
stages are held tighter (they are fp32 transforms of unit-magnitude data).
"""

import numpy as np
import pytest
import torch

import paper_2306_08514_b200 as s
from oracle import srp_oracle as O
from conftest import keep_tags, load_golden, scene_objects, sparse_from_golden
from paper_2306_08514_b200.sampling import spec_offsets

pytestmark = pytest.mark.gpu

MAP_TOL = 1e-4


def np_(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def assert_map_close(z_gpu, z_ref, tol=MAP_TOL):
    err = O.normalized_max_error(np_(z_gpu), z_ref)
    assert np.all(err <= tol), f"normalized max error {err.max():.3e} > {tol:.0e}"
    return err


def assert_argmax_agrees(idx_gpu, z_ref, margin=MAP_TOL):
    idx_gpu = np.atleast_1d(np_(idx_gpu))
    z_ref = np.atleast_2d(z_ref)
    ok = O.peak_margin(z_ref) > margin
    assert np.array_equal(idx_gpu[ok], np.argmax(z_ref, axis=1)[ok])


# ------------------------------------------------------------------ frontend

def test_stft_matches_reference(golden_scene):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    F = g["spectra"].shape[0]
    y = np_(s.stft_frame(g["samples"], frame, range(F)))
    scale = np.abs(g["spectra"]).max(axis=(1, 2), keepdims=True)
    assert np.max(np.abs(y - g["spectra"]) / scale) < 2e-6
    y0 = np_(s.stft_frame(g["samples"], frame, 1))
    assert np.array_equal(y0, y[1])                       # batched == per-frame, bit for bit


def test_fd_gcc_matches_reference(golden_scene):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    psi = np_(s.fd_gcc(g["spectra"], pairs).values)
    d = np.abs(psi - g["psi"])
    assert np.quantile(d, 0.999) < 1e-5 and d.max() < 1e-3
    assert np.allclose(np.abs(psi), 1.0, atol=1e-5)       # PHAT: unit magnitude
    raw = np_(s.fd_gcc(g["spectra"], pairs, weighting="none").values)
    rel = np.abs(raw - g["psi_none"]) / np.abs(g["psi_none"]).max()
    assert rel.max() < 1e-6
    one = s.fd_gcc(g["spectra"][0], pairs)
    assert one.values.shape == (pairs.num_pairs * frame.num_bins,)
    assert np.array_equal(np_(one.values), psi[0])


def test_fused_gcc_frames(golden_scene):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    F = g["psi"].shape[0]
    psi = np_(s.gcc_frames(g["samples"], frame, pairs, range(F)).values)
    d = np.abs(psi - g["psi"])
    assert np.quantile(d, 0.999) < 2e-5 and d.max() < 2e-3


def test_td_gcc_samples_matches_reference(golden_scene):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    gcc = s.FdGcc(torch.from_numpy(g["psi"].astype(np.complex64)).cuda(), pairs.num_pairs,
                  frame.num_bins, "phat")
    for path in ("ifft", "matrix"):
        xi = np_(s.td_gcc_samples(gcc, spec, path).values)
        ref = g["xi_ifft"] if path == "ifft" else g["xi_matrix"]
        err = np.abs(xi - ref).max(axis=1) / np.abs(ref).max(axis=1)
        assert err.max() < 1e-5
    with pytest.raises(ValueError):
        s.td_gcc_samples(gcc, spec, "dft")


def test_fused_frames_to_samples(golden_scene):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    F = g["psi"].shape[0]
    xi = np_(s.frames_to_samples(g["samples"], frame, pairs, spec, range(F)).values)
    err = np.abs(xi - g["xi_ifft"]).max(axis=1) / np.abs(g["xi_ifft"]).max(axis=1)
    assert err.max() < 2e-5
    y = s.stft_frame(g["samples"], frame, range(F))
    xi2 = np_(s.spectra_to_samples(y, pairs, spec).values)
    err2 = np.abs(xi2 - g["xi_ifft"]).max(axis=1) / np.abs(g["xi_ifft"]).max(axis=1)
    assert err2.max() < 2e-5


@pytest.mark.parametrize("kernel", ["warp", "task", "block"])
def test_frontend_kernels_agree(golden_scene, kernel):
    """Every frontend kernel (warp per frame, warp per task, block) meets the golden
    vectors on every output layout: psi, frame-major / lag-major xi, bf16 planes."""
    from paper_2306_08514_b200.frontend import frontend_kernel
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    F = g["psi"].shape[0]
    x = torch.from_numpy(g["samples"].astype(np.float32)).cuda()
    with frontend_kernel(kernel):
        psi = np_(s.gcc_frames(x, frame, pairs, range(F)).values)
        raw = np_(s.gcc_frames(x, frame, pairs, range(F), weighting="none").values)
        xi = s.frames_to_samples(x, frame, pairs, spec, range(F))
        xp = s.frames_to_samples(x, frame, pairs, spec, range(F), planes=True)
        xn = s.frames_to_samples(x, frame, pairs, spec, range(F), planes=True, natural=True)
        one = s.frames_to_samples(x, frame, pairs, spec, 1)
    d = np.abs(psi - g["psi"])
    assert np.quantile(d, 0.999) < 2e-5 and d.max() < 2e-3
    rel = np.abs(raw - g["psi_none"]) / np.abs(g["psi_none"]).max()
    assert rel.max() < 2e-6
    for t in (xi, xp, xn):
        v = np_(t.values)
        err = np.abs(v - g["xi_ifft"]).max(axis=1) / np.abs(g["xi_ifft"]).max(axis=1)
        assert err.max() < 2e-5, f"{kernel}: xi error {err.max():.2e}"
    assert np.array_equal(np_(one.values), np_(xi.values)[1])
    ref, _, _ = s.maps.sample_planes(s.TdGccSamples(xp.values.clone(), spec), spec.total_samples)
    assert torch.equal(xp.bf16_planes.view(torch.int16), ref.view(torch.int16))
    refn, _, _ = s.maps.sample_planes(s.TdGccSamples(xn.values.clone(), spec), spec.total_samples,
                                      natural=spec_offsets(spec))
    S = spec.total_samples
    assert torch.equal(xn.bf16_planes[:, :S, :F].view(torch.int16), refn[:, :S, :F].view(torch.int16))


def test_fused_sspi_chain(golden_scene):
    """frames_to_sspi_map (frontend + SSPI map + argmax in one kernel, xi in shared memory)
    against the reference maps, the unfused chain, argmax-only output and single frames."""
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    F = g["psi"].shape[0]
    x = torch.from_numpy(g["samples"].astype(np.float32)).cuda()
    xi = s.frames_to_samples(x, frame, pairs, spec, range(F))
    for tag in keep_tags(g):
        sp = sparse_from_golden(g, tag)
        z, idx = s.maps.frames_to_sspi_map(sp, x, frame, pairs, spec, range(F))
        ref = g[f"z_sspi_{tag}"]
        zu, iu = s.sspi_map(sp, xi, argmax=True, engine="band")
        if np.abs(ref).max() == 0:
            assert np.all(np_(z) == 0)
            continue
        assert_map_close(z, ref)
        assert_argmax_agrees(idx, ref)
        assert O.normalized_max_error(np_(z), np_(zu)).max() < 1e-5
        zo, io = s.maps.frames_to_sspi_map(sp, x, frame, pairs, spec, range(F), out_map=False)
        assert zo is None and torch.equal(io, idx)
        z1, i1 = s.maps.frames_to_sspi_map(sp, x, frame, pairs, spec, F - 1)
        assert z1.shape == (grid.num_points,) and torch.equal(z1, z[F - 1]) and int(i1) == int(idx[F - 1])
    with pytest.raises(s.DimensionError):
        s.maps.frames_to_sspi_map(sparse_from_golden(g, keep_tags(g)[0]), x[:-1], frame, pairs, spec)


def test_fused_slri_chain(golden_scene):
    """frames_to_slri_map (frontend + fat.xi + tall.y + argmax in one kernel) against the
    reference SLRI maps and the unfused chain; the fused pipeline matches its own eager run."""
    from paper_2306_08514_b200.pipeline import MapPipeline
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    F = g["psi"].shape[0]
    x = torch.from_numpy(g["samples"].astype(np.float32)).cuda()
    xi = s.frames_to_samples(x, frame, pairs, spec, range(F))
    for r in g["ranks"]:
        lr = s.LowRankInterp(g[f"slri_{r}_tall"], g[f"slri_{r}_fat"], np.zeros(r))
        z, idx = s.maps.frames_to_slri_map(lr, x, frame, pairs, spec, range(F))
        assert_map_close(z, g[f"z_slri_{r}"])
        assert_argmax_agrees(idx, g[f"z_slri_{r}"])
        zu, iu = s.slri_map(lr, xi, argmax=True, engine="simt")
        assert O.normalized_max_error(np_(z), np_(zu)).max() < 1e-5
        zo, io = s.maps.frames_to_slri_map(lr, x, frame, pairs, spec, range(F), out_map=False)
        assert zo is None and torch.equal(io, idx)
    pipe = MapPipeline("slri", lr, frame, pairs, spec, frames=F, engine="fused")
    zp, ip = pipe.run(x)
    assert torch.equal(zp, z) and torch.equal(ip, idx)


@pytest.mark.parametrize("wpf", ["1", "2", "4"])
def test_fused_chains_every_warps_per_frame(wpf):
    """The fused chains with 1, 2 and 4 warps per frame forced (SRPGPU_FUSED_WPF, read once
    per process, hence a child pytest) pass the same golden parity tests."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, SRPGPU_FUSED_WPF=wpf)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_parity.py"), "-m", "gpu",
                        "-k", "fused_sspi_chain or fused_slri_chain or fused_chains_weighting"],
                       env=env, cwd=os.path.dirname(here), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.parametrize("weighting,floor", [("none", None), ("phat", 0.5), ("phat", 0.0)])
def test_fused_chains_weighting_and_floor(golden_scene, weighting, floor):
    """The fused chains honour fd_gcc's weighting / floor arguments (frontend.py:127-160)
    exactly as the unfused frontend + map does."""
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    F = g["psi"].shape[0]
    x = torch.from_numpy(g["samples"].astype(np.float32)).cuda()
    xi = s.frames_to_samples(x, frame, pairs, spec, range(F), weighting=weighting, floor=floor)
    sp = sparse_from_golden(g, [t for t in keep_tags(g) if t != "all"][0])
    z, idx = s.maps.frames_to_sspi_map(sp, x, frame, pairs, spec, range(F), weighting=weighting, floor=floor)
    zu, iu = s.sspi_map(sp, xi, argmax=True, engine="band")
    assert O.normalized_max_error(np_(z), np_(zu)).max() < 1e-5
    r = g["ranks"][0]
    lr = s.LowRankInterp(g[f"slri_{r}_tall"], g[f"slri_{r}_fat"], np.zeros(r))
    z2, i2 = s.maps.frames_to_slri_map(lr, x, frame, pairs, spec, range(F), weighting=weighting, floor=floor)
    zu2, iu2 = s.slri_map(lr, xi, argmax=True, engine="simt")
    assert O.normalized_max_error(np_(z2), np_(zu2)).max() < 1e-5


def test_fused_sspi_pipeline(golden_scene):
    """MapPipeline engine 'fused' (one kernel per replay) matches its eager run and the band chain."""
    from paper_2306_08514_b200.pipeline import MapPipeline
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    F = g["psi"].shape[0]
    tag = [t for t in keep_tags(g) if t != "all"][0]
    sp = sparse_from_golden(g, tag)
    x = torch.from_numpy(g["samples"].astype(np.float32)).cuda()
    pipe = MapPipeline("sspi", sp, frame, pairs, spec, frames=F, engine="fused")
    assert pipe.uses_fused_chain()
    z, idx = pipe.run(x)
    torch.cuda.synchronize()
    z_b, i_b = MapPipeline("sspi", sp, frame, pairs, spec, frames=F, engine="band").run(x)
    assert O.normalized_max_error(np_(z), np_(z_b)).max() < 1e-5
    assert_argmax_agrees(idx, g[f"z_sspi_{tag}"])


# ------------------------------------------------------------------ maps

@pytest.mark.parametrize("engine", ["tc", "tile", "tile_f16", "tile_bf16", "band"])
def test_sspi_and_si_maps(golden_scene, engine):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    xi = s.TdGccSamples(torch.from_numpy(g["xi_ifft"].astype(np.float32)).cuda(), spec)
    for tag in keep_tags(g):
        sp = sparse_from_golden(g, tag)
        z, idx = s.sspi_map(sp, xi, argmax=True, engine=engine)
        ref = g[f"z_sspi_{tag}"]
        if np.abs(ref).max() == 0:
            assert np.all(np_(z) == 0)
            continue
        assert_map_close(z, ref)
        assert_argmax_agrees(idx, ref)
        zo, io = s.sspi_map(sp, xi, argmax=True, out_map=False, engine=engine)
        assert zo is None and torch.equal(io, idx)         # argmax-only output
    interp = s.InterpMatrix(g["interp"], spec)
    z_si = s.si_map(interp, xi, engine=engine)
    assert_map_close(z_si, g["z_si"])
    z_all = s.sspi_map(sparse_from_golden(g, "all"), xi, engine=engine)
    assert torch.equal(z_all, z_si)                        # bitwise, as in the reference


def test_sspi_engines_agree_on_frame_batches(golden_scene):
    """Tensor-core engine: a frame's map does not depend on its batch or tile position,
    matches the band engine within the parity bar, and covers F / J tails of the tiles."""
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    sp = sparse_from_golden(g, keep_tags(g)[0])
    x = np.tile(g["xi_ifft"].astype(np.float32), (70, 1))[:300]   # 3 frame tiles, ragged
    xt = s.TdGccSamples(torch.from_numpy(x).cuda(), spec)
    zt, it = s.sspi_map(sp, xt, argmax=True, engine="tc")
    zb, ib = s.sspi_map(sp, xt, argmax=True, engine="band")
    zg, ig = s.sspi_map(sp, xt, argmax=True, engine="tile")
    zh, ih = s.sspi_map(sp, xt, argmax=True, engine="tile_bf16")
    zf, i_f = s.sspi_map(sp, xt, argmax=True, engine="tile_f16")
    z1 = s.sspi_map(sp, s.TdGccSamples(torch.from_numpy(x[7]).cuda(), spec), engine="tc")
    assert torch.equal(zt[7], z1)
    for eng, zz in (("tile", zg), ("tile_bf16", zh), ("tile_f16", zf)):
        g1 = s.sspi_map(sp, s.TdGccSamples(torch.from_numpy(x[7]).cuda(), spec), engine=eng)
        assert torch.equal(zz[7], g1)
    assert_map_close(zh, O.sspi_map(sp.values, sp.col_indices, sp.row_splits, x.astype(np.float64)))
    ref = O.sspi_map(sp.values, sp.col_indices, sp.row_splits, x.astype(np.float64))
    assert_map_close(zt, ref)
    assert_map_close(zb, ref)
    assert_map_close(zg, ref)
    assert_map_close(zf, ref)
    assert_argmax_agrees(it, ref)
    assert_argmax_agrees(ig, ref)
    assert_argmax_agrees(i_f, ref)
    # fp16x3 carries the same 22 operand bits as 3xTF32: the two FP32-class engines agree far
    # inside the parity bar
    assert O.normalized_max_error(np_(zf), np_(zg).astype(np.float64)).max() < 5e-6


def test_natural_planes_from_frontend(golden_scene):
    """The frontend's natural-lag-order bf16 planes equal the permuted split of its f32 samples."""
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    x = torch.from_numpy(g["samples"].astype(np.float32)).cuda()
    for natural in (False, True):
        xi = s.frames_to_samples(x, frame, pairs, spec, planes=True, natural=natural)
        plain = s.TdGccSamples(xi.values.clone(), spec)
        off = spec_offsets(spec) if natural else None
        ref, _, _ = s.maps.sample_planes(plain, spec.total_samples, natural=off)
        assert xi.planes_natural == natural
        if natural:                                         # lag-major: compare the valid frame columns
            f = xi.values.shape[0]
            assert torch.equal(xi.bf16_planes[:, :spec.total_samples, :f].view(torch.int16),
                               ref[:, :spec.total_samples, :f].view(torch.int16))
        else:
            assert torch.equal(xi.bf16_planes.view(torch.int16), ref.view(torch.int16))
    # TF32 hi / lo planes (3xTF32 gathered-window engine): exactly the split of the f32 samples
    xi = s.frames_to_samples(x, frame, pairs, spec, **s.maps.plane_args("tile"))
    assert xi.planes_tf32 and xi.bf16_planes.dtype == torch.float32
    plain = s.TdGccSamples(xi.values.clone(), spec)
    ref, _, _ = s.maps.sample_planes(plain, spec.total_samples, natural=spec_offsets(spec), tf32=True)
    f, st = xi.values.shape[0], spec.total_samples
    assert torch.equal(xi.bf16_planes[:, :st, :f], ref[:, :st, :f])
    hi, lo = xi.bf16_planes[0, :st, :f], xi.bf16_planes[1, :st, :f]
    assert torch.all((hi.view(torch.int32) & 0x1FFF) == 0) and torch.all((lo.view(torch.int32) & 0x1FFF) == 0)
    nat_cols = torch.from_numpy(s.tiles.natural_columns(spec_offsets(spec))).cuda()
    v = xi.values.t()[nat_cols].double()
    assert torch.all((hi.double() + lo.double() - v).abs() <= v.abs() * 2.0 ** -21)


def test_f16_planes_from_frontend(golden_scene):
    """The frontend's fp16 hi / lo planes (fp16x3 gathered-window engine) are exactly the split
    of its f32 samples, carry >= 21 significant bits, and the auto engine takes them only for
    PHAT-weighted (bounded) samples."""
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    x = torch.from_numpy(g["samples"].astype(np.float32)).cuda()
    xi = s.frames_to_samples(x, frame, pairs, spec, **s.maps.plane_args("tile_f16"))
    assert xi.planes_fmt == "f16" and xi.phat and xi.bf16_planes.dtype == torch.float16
    assert xi.bf16_planes.shape[2] % 64 == 0
    plain = s.TdGccSamples(xi.values.clone(), spec)
    ref, _, _ = s.maps.sample_planes(plain, spec.total_samples, natural=spec_offsets(spec), fmt="f16")
    f, st = xi.values.shape[0], spec.total_samples
    assert torch.equal(xi.bf16_planes[:, :st, :f].view(torch.int16), ref[:, :st, :f].view(torch.int16))
    hi, lo = xi.bf16_planes[0, :st, :f].double(), xi.bf16_planes[1, :st, :f].double()
    nat_cols = torch.from_numpy(s.tiles.natural_columns(spec_offsets(spec))).cuda()
    v = xi.values.t()[nat_cols].double()
    assert torch.all((hi + lo - v).abs() <= torch.clamp(v.abs() * 2.0 ** -21, min=2.0 ** -25))
    assert float(v.abs().max()) <= 2 * (frame.half_len - 1)          # the PHAT bound
    with pytest.raises(ValueError):
        s.frames_to_samples(x, frame, pairs, spec, weighting="none", **s.maps.plane_args("tile_f16"))
    assert s.maps.interp_engine(8192, 240.0, "auto", 4096, True, bounded=True) == "tile_f16"
    assert s.maps.interp_engine(8192, 240.0, "auto", 4096, True, bounded=False) == "tile"
    assert not s.maps._bounded(plain) and s.maps._bounded(xi)


@pytest.mark.parametrize("engine", ["tile", "tile_f16"])
def test_tile_map_stages_and_layouts(golden_scene, engine, monkeypatch):
    """The CTA-pair map's two kernels called one after the other (tile-order map + keys, then
    srpgpu_interp_map_untile) give sspi_map's result bit for bit; and the three tile layouts
    (bisected tiles through the scratch, sector runs / 256 consecutive candidates straight
    into grid order, where the grid size allows them) all match the oracle -- on a grid padded
    to a multiple of 8 candidates too, so that every layout is exercised."""
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    tag = keep_tags(g)[0]
    sp = sparse_from_golden(g, tag)
    x = torch.from_numpy(g["samples"].astype(np.float32)).cuda()
    xi = s.frames_to_samples(x, frame, pairs, spec, **s.maps.plane_args(engine))
    z, idx = s.sspi_map(sp, xi, argmax=True, engine=engine)
    op = s.maps.tile_from_sparse(sp, spec_offsets(spec), fmt=s.maps.TILE_ENGINES[engine])
    gather, untile, z2, keys = s.maps.tile_map_stages(sp, xi, engine)
    gather()
    if untile is not None:
        assert not op.grid_order
        untile()
    torch.cuda.synchronize()
    assert torch.equal(z2, z)
    assert torch.equal(s.maps.decode_keys(keys)[0], idx)
    # the same operator on a grid padded with copies of its last rows to J % 8 == 0: bisected
    # sector runs (slack 0) and contiguous tiles (any slack) store straight into grid order
    j = int(np.asarray(sp.row_splits).shape[0] - 1)
    splits = np.asarray(sp.row_splits)
    lo = int(splits[j - 1])
    for mod in (8, 4):       # J % 8 == 0: runs or contiguous; J % 8 == 4: scratch or contiguous
        pad = (-j) % 8 or 8
        if mod == 4:
            pad += 4
        vals = np.concatenate([np.asarray(sp.values)] + [np.asarray(sp.values)[lo:]] * pad)
        cols = np.concatenate([np.asarray(sp.col_indices)] + [np.asarray(sp.col_indices)[lo:]] * pad)
        spl = np.concatenate([splits, splits[-1] + (np.arange(1, pad + 1) * (int(splits[j]) - lo))])
        ref = O.sspi_map(vals, cols, spl, np_(xi.values).astype(np.float64))
        for slack, contiguous in ((0.0, False), (1e9, True)):
            monkeypatch.setattr(s.maps, "CONTIGUOUS_K_SLACK", slack)
            monkeypatch.setattr(s.maps, "CONTIGUOUS_SHORT_SLACK", slack)
            spp = s.SparseInterp(vals, cols, spl, int(sp.num_cols))
            opp = s.maps.tile_from_sparse(spp, spec_offsets(spec), fmt=s.maps.TILE_ENGINES[engine])
            assert opp.contiguous == contiguous and opp.grid_order == (contiguous or mod == 8)
            zp, ip = s.sspi_map(spp, xi, argmax=True, engine=engine)
            assert zp.shape[1] == j + pad
            assert_map_close(zp, ref)
            assert_argmax_agrees(ip, ref)
            assert O.normalized_max_error(np_(zp[:, :j]), np_(z).astype(np.float64)).max() < 5e-6


@pytest.mark.parametrize("engine", ["tile", "tile_f16"])
def test_localizer_mode_keeps_the_argmax(golden_scene, engine):
    """out_map=False (no map, no tile-order scratch, no untile pass: the bench's locate_only
    line) returns the same per-frame argmax as the map-writing call, bit for bit."""
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    sp = sparse_from_golden(g, keep_tags(g)[0])
    x = torch.from_numpy(g["samples"].astype(np.float32)).cuda()
    xi = s.frames_to_samples(x, frame, pairs, spec, **s.maps.plane_args(engine))
    z, idx = s.sspi_map(sp, xi, argmax=True, engine=engine)
    none, idx2 = s.sspi_map(sp, xi, argmax=True, out_map=False, engine=engine)
    assert none is None and torch.equal(idx, idx2)
    assert torch.equal(idx, torch.argmax(z, dim=1))          # the kernel's first-maximum rule


def test_sspi_tile_and_row_kernels_agree(golden_scene):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    sp = sparse_from_golden(g, keep_tags(g)[0])
    x = np.tile(g["xi_ifft"].astype(np.float32), (12, 1))     # >= 32 frames: tile kernel
    zt = s.sspi_map(sp, s.TdGccSamples(torch.from_numpy(x).cuda(), spec))
    zr = torch.stack([s.sspi_map(sp, s.TdGccSamples(torch.from_numpy(x[f]).cuda(), spec))
                      for f in range(g["xi_ifft"].shape[0])])
    assert torch.equal(zt[:zr.shape[0]], zr)


def test_sspi_empty_operator_and_dimension_error(golden_scene):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    interp = s.InterpMatrix(g["interp"], spec)
    sp0 = s.truncate_sparse(interp, 0)
    z = s.sspi_map(sp0, torch.ones(spec.total_samples, device="cuda"))
    assert torch.count_nonzero(z) == 0
    with pytest.raises(s.DimensionError):
        s.sspi_map(sp0, torch.ones(spec.total_samples + 1, device="cuda"))


@pytest.mark.parametrize("engine", ["tc", "simt"])
def test_slri_map(golden_scene, engine):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    xi = torch.from_numpy(g["xi_ifft"].astype(np.float32)).cuda()
    for r in g["ranks"]:
        lr = s.LowRankInterp(g[f"slri_{r}_tall"], g[f"slri_{r}_fat"], np.zeros(r))
        z, idx = s.slri_map(lr, xi, argmax=True, engine=engine)
        assert_map_close(z, g[f"z_slri_{r}"])
        assert_argmax_agrees(idx, g[f"z_slri_{r}"])
    with pytest.raises(s.DimensionError):
        s.slri_map(lr, torch.zeros(3, device="cuda"))


@pytest.mark.parametrize("engine", ["tc", "simt"])
def test_lr_map(golden_scene, engine):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    psi = torch.from_numpy(g["psi"].astype(np.complex64)).cuda()
    for r in g["ranks"]:
        lr = s.LowRankSrp(g[f"lr_{r}_tall"], g[f"lr_{r}_fat"], np.zeros(r))
        gcc = s.FdGcc(psi, pairs.num_pairs, frame.num_bins, "phat")
        z, idx = s.lr_map(lr, gcc, argmax=True, engine=engine)
        assert_map_close(z, g[f"z_lr_{r}"])
        assert_argmax_agrees(idx, g[f"z_lr_{r}"])


@pytest.mark.parametrize("precision", ["tf32", "fp32"])
def test_conventional_map(golden_scene, precision):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    srp = s.build_srp_matrix(tdoa, frame, max_bytes=1 << 34)
    gcc = s.FdGcc(torch.from_numpy(g["psi"].astype(np.complex64)).cuda(), pairs.num_pairs,
                  frame.num_bins, "phat")
    z, idx = s.srp_map_exact(srp, gcc, precision=precision, argmax=True)
    err = assert_map_close(z, g["z_conv"])
    assert err.max() < (1e-5 if precision == "fp32" else MAP_TOL)
    if precision == "tf32":   # fused producer path: gcc_frames(tf32=True) -> tcgen05 GEMM
        F = g["psi"].shape[0]
        g2 = s.gcc_frames(g["samples"], frame, pairs, range(F), tf32=True)
        z2 = s.srp_map_exact(srp, g2)
        assert_map_close(z2, g["z_conv"])
    assert_argmax_agrees(idx, g["z_conv"])
    z1 = s.srp_map_exact(srp, s.FdGcc(gcc.values[0], gcc.num_pairs, gcc.num_bins, "phat"),
                         precision=precision)
    assert z1.shape == (grid.num_points,)
    with pytest.raises(s.DimensionError):
        s.srp_map_exact(srp, s.FdGcc(gcc.values, gcc.num_pairs + 1, gcc.num_bins, "phat"))


def test_locate_and_argmax_ties(golden_scene):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    i, q = s.locate(torch.from_numpy(g["z_conv"][0].astype(np.float32)).cuda(), grid)
    zf = g["z_conv"][0].astype(np.float32)
    assert i == int(np.argmax(zf))
    np.testing.assert_array_equal(q, grid.points[i])
    tie = torch.tensor([0.0, 5.0, 5.0, 1.0], device="cuda")
    g4 = s.CandidateGrid("nf", np.arange(12.0).reshape(4, 3))
    assert s.locate(tie, g4)[0] == 1
    neg = torch.tensor([[-3.0, -1.0, -1.0, -2.0], [-0.0, 0.0, -5.0, -0.0]], device="cuda")
    assert s.map_argmax(neg).tolist() == [1, 0]
    with pytest.raises(s.DimensionError):
        s.locate(torch.zeros(5, device="cuda"), g4)


def test_full_chain_argmax(golden_scene):
    """samples -> fused GCC+iFFT -> SSPI with fused argmax == reference argmax (margin rule)."""
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    F = g["psi"].shape[0]
    xi = s.frames_to_samples(g["samples"], frame, pairs, spec, range(F))
    tag = keep_tags(g)[-2] if len(keep_tags(g)) > 1 else keep_tags(g)[0]
    z, idx = s.sspi_map(sparse_from_golden(g, tag), xi, argmax=True)
    assert_map_close(z, g[f"z_sspi_{tag}"])
    assert_argmax_agrees(idx, g[f"z_sspi_{tag}"])
    zc, ic = s.srp_map_exact(s.build_srp_matrix(tdoa, frame, max_bytes=1 << 34),
                             s.gcc_frames(g["samples"], frame, pairs, range(F)), argmax=True)
    assert_map_close(zc, g["z_conv"])
    assert_argmax_agrees(ic, g["z_conv"])


# ------------------------------------------------------------------ known answers / edges

def test_known_answers_on_gpu(known):
    # single active bin -> z = 2 cos(w_k dt)   (test_srp.py:56-65)
    frame = s.FrameSpec(frame_len=8, sample_rate=800)
    srp = s.build_srp_matrix(s.TdoaTable(known["ka_cos_dt"], np.array([2e-3])), frame)
    v = torch.zeros(3, dtype=torch.complex64, device="cuda")
    v[0] = 1.0
    z = s.srp_map_exact(srp, s.FdGcc(v, 1, 3, "none"), precision="fp32")
    np.testing.assert_allclose(np_(z), known["ka_cos_z"], atol=1e-6)
    # single bin -> sampled cosine            (test_sampling.py:67-79)
    f32 = s.FrameSpec(frame_len=32, sample_rate=1000)
    spec = s.SampleSpec(known["ka_cos_counts"], 0, 16)
    per = torch.zeros((3, 15), dtype=torch.complex64, device="cuda")
    per[:, 4] = 1.0
    xi = s.td_gcc_samples(s.FdGcc(per.reshape(-1), 3, 15, "none"), spec)
    np.testing.assert_allclose(np_(xi.values), known["ka_cos_xi"], atol=1e-5)
    # integer circular delay -> exact phase ramp (rect window)   (test_frontend.py:89-100)
    arr = s.MicrophoneArray(np.array([[0.0, 0, 0], [0.1, 0, 0]]))
    pairs = s.enumerate_pairs(arr)
    rect = s.FrameSpec(frame_len=32, sample_rate=1000, window="rect")
    psi = s.fd_gcc(s.stft_frame(known["ka_ramp_signal"], rect, 0), pairs)
    np.testing.assert_allclose(np_(psi.values), known["ka_ramp_psi"], atol=2e-6)
    # floored bin is exactly 0                (test_frontend.py:137-145)
    fl = np_(s.fd_gcc(known["ka_floor_spectra"], pairs).values)
    assert fl[4] == 0.0
    np.testing.assert_allclose(np.abs(np.delete(fl, 4)), 1.0, atol=1e-6)
    # explicit floor on all-zero spectra gives 0 (test_frontend.py:102-105)
    zero = s.fd_gcc(np.zeros((2, 9), complex), pairs, floor=1e-9)
    assert torch.count_nonzero(zero.values) == 0


def test_frontend_errors():
    arr = s.MicrophoneArray(np.array([[0.0, 0, 0], [0.1, 0, 0]]))
    pairs = s.enumerate_pairs(arr)
    spec = s.FrameSpec(frame_len=16, sample_rate=100, hop=4)
    x = np.random.default_rng(0).standard_normal((1, 40))
    out = np_(s.stft_frame(x, spec, 2))
    np.testing.assert_allclose(out[0], np.fft.rfft(x[0, 8:24] * s.frame_window(spec)), atol=1e-5)
    assert s.num_frames(spec, 40) == 7
    with pytest.raises(IndexError):
        s.stft_frame(x, spec, 7)
    with pytest.raises(IndexError):
        s.stft_frame(x, spec, -1)
    with pytest.raises(s.DimensionError):
        s.fd_gcc(np.zeros((3, 9), complex), pairs)
    with pytest.raises(ValueError):
        s.fd_gcc(np.zeros((2, 9), complex), pairs, weighting="scot")
    # identical channels give unit phase     (test_frontend.py:83-87)
    y = np.random.default_rng(3).standard_normal(9) + 1j * np.random.default_rng(4).standard_normal(9)
    np.testing.assert_allclose(np_(s.fd_gcc(np.stack([y, y]), pairs).values), 1.0, atol=1e-6)


def test_evaluate_map_dispatch(golden_scene):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    gcc = s.FdGcc(torch.from_numpy(g["psi"].astype(np.complex64)).cuda(), pairs.num_pairs,
                  frame.num_bins, "phat")
    tag = keep_tags(g)[0]
    z = s.evaluate_map("sspi", sparse_from_golden(g, tag), spec, frame, gcc, "auto")
    assert_map_close(z, g[f"z_sspi_{tag}"])
    z = s.evaluate_map("si", s.InterpMatrix(g["interp"], spec), spec, frame, gcc, "matrix")
    assert_map_close(z, g["z_si"])
    with pytest.raises(ValueError):
        s.evaluate_map("xyz", None, spec, frame, gcc, "ifft")


def test_pipeline_graph_matches_eager(golden_scene):
    from paper_2306_08514_b200.pipeline import MapPipeline
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    F = g["psi"].shape[0]
    x = g["samples"][:, :(F - 1) * frame.hop + frame.frame_len]
    tag = keep_tags(g)[0]
    sp = sparse_from_golden(g, tag)
    xi = s.frames_to_samples(x, frame, pairs, spec, range(F))
    eng = s.maps.map_engine("sspi", sp, "auto", F)
    pipe = MapPipeline("sspi", sp, frame, pairs, spec, frames=F, engine=eng)   # the unfused chain
    z, idx = pipe.run(x)
    z2, idx2 = s.sspi_map(sp, xi, argmax=True, engine=eng)
    assert torch.equal(z, z2) and torch.equal(idx, idx2)
    auto = MapPipeline("sspi", sp, frame, pairs, spec, frames=F)               # fused where eligible
    za, ia = auto.run(x)
    assert O.normalized_max_error(np_(za), np_(z2)).max() < 1e-5
    assert_argmax_agrees(ia, g[f"z_sspi_{tag}"])
    conv = MapPipeline("conv", s.build_srp_matrix(tdoa, frame, max_bytes=1 << 34), frame, pairs,
                       frames=F)
    zc, ic = conv.run(torch.from_numpy(x.astype(np.float32)).cuda())
    assert_map_close(zc, g["z_conv"])
    assert_argmax_agrees(ic, g["z_conv"])


def test_band_group_placement_bit_identical(golden_scene):
    """Placing candidate groups in another order leaves every map bit-identical
    (tile kernel and the small-batch rows kernel both read the slot meta)."""
    from paper_2306_08514_b200 import maps
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    sp = sparse_from_golden(g, keep_tags(g)[0])
    j = sp.row_splits.shape[0] - 1
    rows = np.repeat(np.arange(j), np.diff(sp.row_splits))
    groups = (j + 3) // 4
    for nf in (g["psi"].shape[0], 40):
        n = (nf - 1) * frame.hop + frame.frame_len
        x = np.tile(g["samples"], (1, n // g["samples"].shape[1] + 1))[:, :n]
        xi = s.frames_to_samples(x, frame, pairs, spec, range(nf))
        out = []
        for placement in (None, np.arange(groups)[::-1].copy()):
            op = maps.BandOperator(rows, sp.col_indices, sp.values, j, int(sp.num_cols),
                                   spec.offsets, placement=placement)
            out.append(maps._band_map(op, xi, True, True))
        assert torch.equal(out[0][0], out[1][0]) and torch.equal(out[0][1], out[1][1])


def test_map_stream_matches_pipeline(golden_scene):
    """Streamed batches (overlapped copies, rotating slots) give the pipeline's argmax."""
    from paper_2306_08514_b200.pipeline import MapPipeline, MapStream
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    F = 4
    n = (F - 1) * frame.hop + frame.frame_len
    sp = sparse_from_golden(g, keep_tags(g)[0])
    total = g["samples"].shape[1]
    starts = [0, frame.hop, 2 * frame.hop, 5 * frame.hop, frame.hop]
    starts = [st for st in starts if st + n <= total]
    batches = [torch.from_numpy(np.ascontiguousarray(g["samples"][:, st:st + n], dtype=np.float32))
               .pin_memory() for st in starts]
    ref = MapPipeline("sspi", sp, frame, pairs, spec, frames=F)
    want = [ref.run(b)[1].cpu().numpy() for b in batches]
    stream = MapStream("sspi", sp, frame, pairs, spec, frames=F, depth=2)
    got = []
    for t, b in enumerate(batches):
        assert stream.submit(b) == t
        if t > 0:
            got.append(stream.result(t - 1))      # previous batch, while batch t is in flight
    got.append(stream.result(len(batches) - 1))
    for t in range(len(batches)):
        assert np.array_equal(got[t], want[t])
    with pytest.raises(ValueError):
        stream.submit(batches[0][:, :-1])
    with pytest.raises(ValueError):
        stream.result(len(batches))               # not submitted yet
    for t in range(2):                            # rotate both slots past batch 0
        stream.submit(batches[0])
    with pytest.raises(ValueError):
        stream.result(0)                          # slot already reused


def test_conventional_map_onchip_steering(golden_scene):
    """H generated on chip from the TDOA table (no stored operator) matches the reference map."""
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    op = s.steering_operator(tdoa, frame)
    F = g["psi"].shape[0]
    gcc = s.gcc_frames(g["samples"], frame, pairs, range(F), tf32=True)
    z, idx = s.srp_map_exact(op, gcc, argmax=True)
    assert_map_close(z, g["z_conv"])
    assert_argmax_agrees(idx, g["z_conv"])
    gcc2 = s.FdGcc(torch.from_numpy(g["psi"].astype(np.complex64)).cuda(), pairs.num_pairs,
                   frame.num_bins, "phat")
    assert_map_close(s.srp_map_exact(op, gcc2), g["z_conv"])
    err = assert_map_close(s.srp_map_exact(op, gcc2, precision="tf32x3"), g["z_conv"])
    assert err.max() < 1e-5                      # split precision: fp32 class
    with pytest.raises(ValueError):
        s.srp_map_exact(op, gcc2, precision="fp32")
    with pytest.raises(ValueError):
        s.srp_map_exact(op, gcc, precision="tf32x3")   # pre-rounded psi cannot be split
