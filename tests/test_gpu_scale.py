"""GPU parity at the BASELINE.json configurations' full grids (cfg2, cfg3, cfg4).

Frame counts are reduced where the float64 oracle would take too long; the
checks are size-independent: per-frame normalized max error <= 1e-4 against the
oracle on a frame subset, argmax agreement on margin-qualified frames, bitwise
invariance of the maps under frame partitioning (the multi-GPU split), and the
nnz / rank sweeps of BASELINE configs[1].
"""

import numpy as np
import pytest
import torch

import paper_2306_08514_b200 as s
from paper_2306_08514_b200 import workloads
from paper_2306_08514_b200.operators import low_rank_interp_from_svd, low_rank_srp_from_svd
from oracle import srp_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-4


def oracle_psi(wl, nf):
    win = O.frame_window(wl.frame.frame_len, wl.frame.window)
    spectra = O.stft_frames(wl.samples.astype(np.float64), wl.frame.frame_len, wl.frame.hop, win,
                            np.arange(nf))
    return O.fd_gcc(spectra, wl.pairs.pairs)


def check(z_gpu, z_ref, idx_gpu=None):
    z = z_gpu.detach().float().cpu().numpy()[: z_ref.shape[0]]
    err = O.normalized_max_error(z, z_ref)
    assert err.max() <= TOL, f"normalized max error {err.max():.3e}"
    if idx_gpu is not None:
        ok = O.peak_margin(z_ref) > TOL
        idx = idx_gpu.cpu().numpy()[: z_ref.shape[0]]
        assert np.array_equal(idx[ok], np.argmax(z_ref, axis=1)[ok])
    return float(err.max())


@pytest.fixture(scope="module")
def cfg2():
    wl = workloads.make("cfg2")
    x = torch.from_numpy(wl.samples).cuda()
    xi = s.frames_to_samples(x, wl.frame, wl.pairs, wl.spec)
    psi_ref = oracle_psi(wl, 32)
    xi_ref = O.td_gcc_samples(psi_ref, wl.spec.counts, wl.frame.half_len)
    return wl, x, xi, psi_ref, xi_ref


def test_cfg2_samples_and_sspi_global_fit(cfg2):
    wl, x, xi, psi_ref, xi_ref = cfg2
    got = xi.values[:32].cpu().numpy()
    err = np.abs(got - xi_ref).max(axis=1) / np.abs(xi_ref).max(axis=1)
    assert err.max() < 2e-5
    interp = s.build_interp_matrix(wl.tdoa, wl.spec, wl.frame)
    sp = s.truncate_sparse(interp, 2 * wl.grid.num_points * wl.pairs.num_pairs)
    z, idx = s.sspi_map(sp, xi, argmax=True)
    z_ref = O.sspi_map(sp.values, sp.col_indices, sp.row_splits, xi_ref)
    check(z, z_ref, idx)
    # frame partition (the multi-GPU split) leaves every map bit-identical
    half = wl.num_frames // 2
    xa = s.frames_to_samples(x, wl.frame, wl.pairs, wl.spec, range(0, half))
    xb = s.frames_to_samples(x, wl.frame, wl.pairs, wl.spec, range(half, wl.num_frames))
    za, ia = s.sspi_map(sp, xa, argmax=True)
    zb, ib = s.sspi_map(sp, xb, argmax=True)
    assert torch.equal(torch.cat([za, zb]), z) and torch.equal(torch.cat([ia, ib]), idx)


@pytest.mark.parametrize("nnz", [1, 2, 4, 8, 16])
def test_cfg2_sspi_nnz_sweep(cfg2, nnz):
    wl, x, xi, psi_ref, xi_ref = cfg2
    fx = s.sparse_interp_fixed(wl.tdoa, wl.spec, wl.frame, nnz)
    z, idx = s.sspi_map(fx, xi, argmax=True)
    csr = fx.to_csr()
    z_ref = O.sspi_map(csr.values, csr.col_indices, csr.row_splits, xi_ref)
    check(z, z_ref, idx)


def test_cfg2_rank_sweeps(cfg2):
    wl, x, xi, psi_ref, xi_ref = cfg2
    interp = s.build_interp_matrix(wl.tdoa, wl.spec, wl.frame)
    u, sv, vt = np.linalg.svd(interp.matrix, full_matrices=False)
    srp = s.build_srp_matrix(wl.tdoa, wl.frame)
    hu, hs, hvt = np.linalg.svd(srp.matrix, full_matrices=False)
    gcc = s.gcc_frames(x, wl.frame, wl.pairs)
    for r in (1, 2, 4, 8, 16, 32):
        lri = low_rank_interp_from_svd(u, sv, vt, r)
        z, idx = s.slri_map(lri, xi, argmax=True)
        check(z, O.slri_map(lri.tall, lri.fat, xi_ref), idx)
        lrs = low_rank_srp_from_svd(hu, hs, hvt, r)
        z, idx = s.lr_map(lrs, gcc, argmax=True)
        check(z, O.lr_map(lrs.tall, lrs.fat, psi_ref), idx)


def test_cfg2_conventional(cfg2):
    wl, x, xi, psi_ref, xi_ref = cfg2
    srp = s.build_srp_matrix(wl.tdoa, wl.frame)
    z_ref = O.srp_map_exact(srp.matrix, psi_ref)
    for prec in ("tf32", "fp32"):
        gcc = s.gcc_frames(x, wl.frame, wl.pairs, tf32=(prec == "tf32"))
        z, idx = s.srp_map_exact(srp, gcc, precision=prec, argmax=True)
        check(z, z_ref, idx)


def test_cfg2_fused_chains_and_splitk(cfg2):
    """The bench's headline path at full batch (1000 frames, one fused kernel per step) for
    SSPI (global 2JP fit) and SLRI (R = 16), and the split-K on-chip conventional map,
    against the float64 oracle on the first 32 frames."""
    from paper_2306_08514_b200.pipeline import MapPipeline
    wl, x, xi, psi_ref, xi_ref = cfg2
    interp = s.build_interp_matrix(wl.tdoa, wl.spec, wl.frame)
    sp = s.truncate_sparse(interp, s.resolve_sparsity("2jp", wl.grid.num_points, wl.pairs.num_pairs,
                                                      interp.matrix.size))
    lr = s.truncate_low_rank(interp, 16)
    F = wl.num_frames
    n = (F - 1) * wl.frame.hop + wl.frame.frame_len
    for variant, op, z_ref in (
            ("sspi", sp, O.sspi_map(sp.values, sp.col_indices, sp.row_splits, xi_ref)),
            ("slri", lr, O.slri_map(lr.tall, lr.fat, xi_ref))):
        pipe = MapPipeline(variant, op, wl.frame, wl.pairs, wl.spec, frames=F)
        assert pipe.uses_fused_chain()
        z, idx = pipe.run(x[:, :n])
        torch.cuda.synchronize()
        check(z, z_ref, idx)
    steer = s.steering_operator(wl.tdoa, wl.frame)
    gcc = s.gcc_frames(x, wl.frame, wl.pairs, tf32=True)
    z, idx = s.srp_map_exact(steer, gcc, argmax=True)          # 56 output tiles -> 2 K slices
    check(z, O.srp_map_exact(s.build_srp_matrix(wl.tdoa, wl.frame).matrix, psi_ref), idx)


@pytest.fixture(scope="module")
def cfg3():
    wl = workloads.make("cfg3", num_frames=256)
    x = torch.from_numpy(wl.samples).cuda()
    psi_ref = oracle_psi(wl, 8)
    xi_ref = O.td_gcc_samples(psi_ref, wl.spec.counts, wl.frame.half_len)
    return wl, x, psi_ref, xi_ref


@pytest.mark.parametrize("engine", ["tc", "band"])
def test_cfg3_full_grid(cfg3, engine):
    wl, x, psi_ref, xi_ref = cfg3
    assert wl.grid.num_points == 32760 and wl.pairs.num_pairs == 28
    xi = s.frames_to_samples(x, wl.frame, wl.pairs, wl.spec, planes=(engine == "tc"))
    interp = s.build_interp_matrix(wl.tdoa, wl.spec, wl.frame)
    sp = s.truncate_sparse(interp, 2 * wl.grid.num_points * wl.pairs.num_pairs)
    z, idx = s.sspi_map(sp, xi, argmax=True, engine=engine)
    check(z, O.sspi_map(sp.values, sp.col_indices, sp.row_splits, xi_ref), idx)
    lr = s.truncate_low_rank(interp, 16)
    z, idx = s.slri_map(lr, xi, argmax=True, engine="tc" if engine == "tc" else "simt")
    check(z, O.slri_map(lr.tall, lr.fat, xi_ref), idx)
    # pole rows (polar 180 deg, 360 azimuths) are exact duplicates -> identical map values
    zz = z[:, -360:]
    assert torch.equal(zz, zz[:, :1].expand_as(zz))


def test_cfg3_conventional_tf32(cfg3):
    wl, x, psi_ref, xi_ref = cfg3
    srp = s.build_srp_matrix(wl.tdoa, wl.frame, max_bytes=1 << 34)
    gcc = s.gcc_frames(x, wl.frame, wl.pairs, tf32=True)
    z_ref = O.srp_map_exact(srp.matrix, psi_ref)
    z, idx = s.srp_map_exact(srp, gcc, argmax=True)
    check(z, z_ref, idx)
    z2, idx2 = s.srp_map_exact(s.steering_operator(wl.tdoa, wl.frame), gcc, argmax=True)
    check(z2, z_ref, idx2)


def test_cfg4_conventional_onchip_steering():
    """cfg4's H (164 GB as fp32) is never stored: generated on chip; oracle on a row block.

    3xTF32 (split-precision tensor-core GEMM) meets the 1e-4 bound; plain TF32 is
    allowed at cfg4 by BASELINE.json "with error reported" and is only bounded loosely.
    """
    wl = workloads.make("cfg4", num_frames=8)
    x = torch.from_numpy(wl.samples).cuda()
    op = s.steering_operator(wl.tdoa, wl.frame)
    z, idx = s.srp_map_exact(op, s.gcc_frames(x, wl.frame, wl.pairs), precision="tf32x3", argmax=True)
    z_tf32 = s.srp_map_exact(op, s.gcc_frames(x, wl.frame, wl.pairs, tf32=True))
    psi_ref = oracle_psi(wl, 2)
    # oracle rows: a 1/97 subsample plus each frame's peak neighbourhood, so that the
    # normalization max|z_ref| is the map's true maximum (the north-star metric)
    peaks = idx[:2].cpu().numpy()
    near = np.concatenate([np.arange(max(0, q - 300), min(wl.grid.num_points, q + 300)) for q in peaks])
    rows = np.unique(np.concatenate([np.arange(0, wl.grid.num_points, 97), near]))
    sub = s.TdoaTable(wl.tdoa.delta_t[rows], wl.tdoa.limits)
    H = s.build_srp_matrix(sub, wl.frame, max_bytes=1 << 34).matrix
    z_ref = O.srp_map_exact(H, psi_ref)
    got = z[:2, rows].float().cpu().numpy()
    err = O.normalized_max_error(got, z_ref)
    assert err.max() <= TOL
    err_tf32 = O.normalized_max_error(z_tf32[:2, rows].float().cpu().numpy(), z_ref)
    print(f"cfg4 conventional: 3xTF32 error {err.max():.2e}, TF32 error {err_tf32.max():.2e}")
    assert err_tf32.max() <= 2e-3
    # the peak itself: the GPU argmax is (one of) the oracle's maxima over the checked rows
    for f in range(2):
        j = int(np.searchsorted(rows, peaks[f]))
        assert z_ref[f, j] >= z_ref[f].max() * (1 - 2 * TOL)


@pytest.fixture(scope="module")
def cfg4_fit():
    wl = workloads.make("cfg4", num_frames=64)
    return wl, s.sparse_interp_fixed(wl.tdoa, wl.spec, wl.frame, 2)


@pytest.mark.parametrize("engine", ["tile", "tile_f16", "tile_bf16", "band"])
def test_cfg4_full_grid_sspi(cfg4_fit, engine):
    wl, fx = cfg4_fit
    assert wl.grid.num_points == 334611 and wl.pairs.num_pairs == 120
    x = torch.from_numpy(wl.samples).cuda()
    xi = s.frames_to_samples(x, wl.frame, wl.pairs, wl.spec, **s.maps.plane_args(engine))
    z, idx = s.sspi_map(fx, xi, argmax=True, engine=engine)
    nf = 4
    xi_ref = O.td_gcc_samples(oracle_psi(wl, nf), wl.spec.counts, wl.frame.half_len)
    z_ref = np.zeros((nf, wl.grid.num_points))
    for p in range(wl.pairs.num_pairs):
        k = int(fx.kept[p])
        z_ref += np.einsum("jk,fjk->fj", fx.values[p, :, :k], xi_ref[:, fx.cols[p, :, :k]])
    check(z, z_ref, idx)


@pytest.fixture(scope="module")
def cfg4_global():
    """The bench headline's operator: cfg4 SSPI with the reference's global top-Q rule at
    Q = 2JP (interpolation.py:155-175), streamed (the dense 18.7 GB Lambda is never built)."""
    wl = workloads.make("cfg4", num_frames=300)
    j, p = wl.grid.num_points, wl.pairs.num_pairs
    keep = s.resolve_sparsity("2jp", j, p, j * wl.spec.total_samples)
    return wl, s.truncate_sparse_streamed(wl.tdoa, wl.spec, wl.frame, keep)


def _csr_rows(sp, rows):
    """The CSR rows `rows` of a SparseInterp (oracle on a row block)."""
    splits = np.asarray(sp.row_splits)
    lo, hi = splits[rows], splits[rows + 1]
    idx = np.concatenate([np.arange(a, b) for a, b in zip(lo, hi)])
    sub_splits = np.concatenate([[0], np.cumsum(hi - lo)])
    return np.asarray(sp.values)[idx], np.asarray(sp.col_indices)[idx], sub_splits


@pytest.mark.parametrize("engine", ["auto", "tile", "tile_bf16"])
def test_cfg4_global_fit_pipeline(cfg4_global, engine):
    """The default bench path: MapPipeline (CUDA graph: fused frontend -> fp16x3 (auto, PHAT) or
    3xTF32 gathered-window map on CTA pairs -> argmax) at cfg4 with the global fit, 300 frames (two unit frame
    tiles + a ragged one), against the float64 oracle on a row block: a 1/61 subsample plus
    each checked frame's peak neighbourhood, so max|z_ref| is the map's true maximum."""
    from paper_2306_08514_b200.pipeline import MapPipeline
    wl, sp = cfg4_global
    assert wl.grid.num_points == 334611 and sp.num_kept == 2 * 334611 * 120
    pipe = MapPipeline("sspi", sp, wl.frame, wl.pairs, wl.spec, frames=wl.num_frames, engine=engine)
    assert not pipe.uses_fused_chain()
    if engine == "auto":
        assert s.maps.map_engine("sspi", sp, "auto", wl.num_frames) == "tile"
        assert s.maps.map_engine("sspi", sp, "auto", wl.num_frames, bounded=True) == "tile_f16"
    z, idx = pipe.run(torch.from_numpy(wl.samples).cuda())
    torch.cuda.synchronize()
    nf = 3
    frames = np.array([0, 1, wl.num_frames - 1])                   # last frame: the ragged unit
    x64 = wl.samples.astype(np.float64)
    win = O.frame_window(wl.frame.frame_len, wl.frame.window)
    psi = O.fd_gcc(O.stft_frames(x64, wl.frame.frame_len, wl.frame.hop, win, frames), wl.pairs.pairs)
    xi_ref = O.td_gcc_samples(psi, wl.spec.counts, wl.frame.half_len)
    peaks = idx[frames].cpu().numpy()
    near = np.concatenate([np.arange(max(0, q - 400), min(wl.grid.num_points, q + 400)) for q in peaks])
    rows = np.unique(np.concatenate([np.arange(0, wl.grid.num_points, 61), near]))
    vals, cols, splits = _csr_rows(sp, rows)
    z_ref = O.sspi_map(vals, cols, splits, xi_ref)
    got = z[frames][:, rows].float().cpu().numpy()
    err = O.normalized_max_error(got, z_ref)
    assert err.max() <= TOL
    if engine in ("auto", "tile"):
        assert err.max() <= 2e-6, f"split operands with fp32 folds: FP32-class error expected, got {err.max():.2e}"
    for k in range(nf):       # the GPU argmax is the oracle's maximum over the checked rows
        j = int(np.searchsorted(rows, peaks[k]))
        assert z_ref[k, j] >= z_ref[k].max() * (1 - 2 * TOL)
    # the map does not depend on the batch: a frame's row equals its single-frame map
    eng1 = s.maps.map_engine("sspi", sp, engine, 1, bounded=True)      # the pipeline weights with PHAT
    xi1 = s.frames_to_samples(torch.from_numpy(wl.samples).cuda(), wl.frame, wl.pairs, wl.spec, range(1, 2),
                              **s.maps.plane_args(eng1))
    z1 = s.sspi_map(sp, xi1, engine=eng1)
    assert torch.equal(z1[0], z[1])
    print(f"cfg4 global fit ({engine}): normalized max error {err.max():.2e} over {rows.size} rows")


def _combine(keys_list):
    """The all-reduce MAX of candidate_partition, in one process."""
    from paper_2306_08514_b200 import distributed as D
    k = D.keys_to_signed(keys_list[0].clone())
    for other in keys_list[1:]:
        k = torch.maximum(k, D.keys_to_signed(other))
    return D.decode_host_keys(D.signed_to_keys(k))


def test_candidate_partition_conventional_ties():
    """Candidate partition (srp.py:71: rows are independent): two row blocks of the on-chip
    conventional map, their kernel argmax re-based to global indices and MAX-combined, give
    the full map's first maximum -- including a tie planted across the block boundary (rows
    J/2 - 1 and J/2 copy the peak row's TDOAs, so three rows share the maximum bitwise)."""
    from paper_2306_08514_b200 import distributed as D
    from paper_2306_08514_b200.pipeline import MapPipeline
    wl = workloads.make("cfg2", num_frames=4096)          # >= 148 output tiles: no split-K
    x = torch.from_numpy(wl.samples).cuda()
    j = wl.grid.num_points
    op = s.steering_operator(wl.tdoa, wl.frame)
    pipe = MapPipeline("conv", op, wl.frame, wl.pairs, wl.spec, frames=wl.num_frames)
    z0, i0 = pipe.run(x)
    peak = int(i0[0])
    dt = wl.tdoa.delta_t.copy()
    dt[j // 2 - 1] = dt[peak]
    dt[j // 2] = dt[peak]
    op2 = s.steering_operator(s.TdoaTable(dt, wl.tdoa.limits), wl.frame)
    full = MapPipeline("conv", op2, wl.frame, wl.pairs, wl.spec, frames=wl.num_frames)
    zf, idf = full.run(x)
    zf, idf = zf.clone(), idf.clone()
    keys = []
    for r in range(2):
        sh = D.CandidateShard("conv", op2, wl.frame, wl.pairs, wl.spec, wl.num_frames, r, 2)
        sh.pipe.run(x)
        z_b, _ = sh.pipe.z, sh.pipe.index
        assert torch.equal(z_b, zf[:, sh.first:sh.first + sh.count])        # row-local: bitwise
        keys.append(sh.step())
    idx, val = _combine(keys)
    zc = zf.cpu().numpy()
    assert np.array_equal(idx.cpu().numpy(), np.argmax(zc, axis=1))        # first maximum, ties
    assert np.array_equal(idx.cpu().numpy(), idf.cpu().numpy())
    assert int(idx[0]) == min(peak, j // 2 - 1)
    assert np.array_equal(val.cpu().numpy(), zc.max(axis=1))


def test_candidate_partition_cfg4_sspi(cfg4_global):
    """The largest grid split by candidates (cfg4, global fit, 3xTF32 gathered windows):
    two row blocks + the key MAX give the full map's argmax on every margin-qualified frame."""
    from paper_2306_08514_b200 import distributed as D
    from paper_2306_08514_b200.pipeline import MapPipeline
    wl, sp = cfg4_global
    x = torch.from_numpy(wl.samples).cuda()
    zf, idf = MapPipeline("sspi", sp, wl.frame, wl.pairs, wl.spec, frames=wl.num_frames).run(x)
    zf, idf = zf.clone(), idf.clone()
    keys = []
    for r in range(2):
        sh = D.CandidateShard("sspi", sp, wl.frame, wl.pairs, wl.spec, wl.num_frames, r, 2)
        sh.pipe.run(x)
        keys.append(sh.step())
        del sh
    idx, val = _combine(keys)
    z = zf.cpu().numpy()
    part = np.partition(z, -2, axis=1)
    ok = (part[:, -1] - part[:, -2]) / np.abs(z).max(axis=1) > TOL
    assert ok.sum() > wl.num_frames // 2
    assert np.array_equal(idx.cpu().numpy()[ok], idf.cpu().numpy()[ok])
