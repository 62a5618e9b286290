"""Host-side logic of the product (no GPU): geometry, operator fits, band layout.

Operator fitting stays on the host and is uploaded once; these tests pin it
bit-exactly to reference-generated golden vectors (sparse structure, TDOA,
lag counts) and check the tiled-band operator encoding decodes back to the
reference CSR exactly.
"""

import numpy as np
import pytest
from numpy.testing import assert_allclose, assert_array_equal

import paper_2306_08514_b200 as s
from paper_2306_08514_b200 import operators, scene
from paper_2306_08514_b200.distributed import decode_host_keys, offset_keys, partition
from conftest import keep_tags, scene_objects, sparse_from_golden


def test_scene_matches_reference(golden_scene):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    assert_array_equal(pairs.pairs, g["pairs"])
    assert_array_equal(pairs.distances, g["distances"])
    assert_array_equal(tdoa.delta_t, g["delta_t"])
    assert_array_equal(tdoa.limits, g["limits"])
    assert_array_equal(spec.counts, g["counts"])
    assert_array_equal(spec.offsets, g["offsets"])
    assert_array_equal(s.frame_window(frame), g["window"])


def test_grids():
    g = s.build_nf_grid((0, 0, 0), (4, 4, 0), 0.1)
    assert g.num_points == 1681
    assert_allclose(g.points[1], [0.1, 0, 0])          # x fastest
    ff = s.build_ff_grid(1.0, collapse_poles=False)
    assert ff.num_points == 32760
    assert np.all(ff.points[-360:] == np.array([0.0, 0.0, -1.0]))
    assert s.build_ff_grid(1.0).num_points == 32401      # reference layout (pole once)
    big = s.build_nf_grid((0, 0, 0), (4, 4, 2.5), 0.05)
    assert big.num_points == 334611


def test_operators_match_reference(golden_scene):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    interp = s.build_interp_matrix(tdoa, spec, frame)
    assert_array_equal(interp.matrix, g["interp"])
    for tag in keep_tags(g):
        sp = s.truncate_sparse(interp, int(g[f"sp_{tag}_keep"]))
        ref = sparse_from_golden(g, tag)
        assert_array_equal(sp.values, ref.values)
        assert_array_equal(sp.col_indices, ref.col_indices)
        assert_array_equal(sp.row_splits, ref.row_splits)
    srp = s.build_srp_matrix(tdoa, frame, max_bytes=1 << 34)
    z = 2.0 * (g["psi"] @ srp.matrix.T).real
    assert_allclose(z, g["z_conv"], rtol=1e-12, atol=1e-9)


def test_truncate_sparse_ties_and_bounds():
    mk = lambda m: s.InterpMatrix(np.asarray(m, float), s.SampleSpec(np.zeros(np.shape(m)[1], np.int64), 0, 64))
    sp = s.truncate_sparse(mk([[0.5, -0.5], [0.5, 0.5]]), 2)
    assert_array_equal(sp.to_dense(), [[0.5, -0.5], [0.0, 0.0]])
    sp = s.truncate_sparse(mk([[0.9, -0.5, 0.1], [0.2, -0.8, 0.3]]), 2)
    assert_array_equal(sp.to_dense(), [[0.9, 0, 0], [0, -0.8, 0]])
    assert s.truncate_sparse(mk([[1.0, 2.0]]), 0).num_kept == 0
    with pytest.raises(ValueError):
        s.truncate_sparse(mk([[1.0, 2.0]]), 3)
    with pytest.raises(ValueError):
        s.truncate_sparse(mk([[1.0, 2.0]]), -1)


def test_fixed_nnz_fit_keeps_nearest_lags(golden_scene):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    interp = s.build_interp_matrix(tdoa, spec, frame)
    off = spec.offsets
    for nnz in (1, 2, 4):
        sp = s.truncate_sparse_fixed(interp, nnz)
        expect = sum(min(nnz, int(2 * c + 1)) for c in spec.counts) * grid.num_points
        assert sp.num_kept == expect
        dense = sp.to_dense()
        kept = np.zeros(interp.matrix.shape, bool)
        kept[np.repeat(np.arange(grid.num_points), np.diff(sp.row_splits)), sp.col_indices] = True
        mag = np.abs(interp.matrix)
        for p in range(spec.num_pairs):
            blk, kb = mag[:, off[p]:off[p + 1]], kept[:, off[p]:off[p + 1]]
            lo = np.where(kb, blk, np.inf).min(axis=1)
            hi = np.where(kb, -np.inf, blk).max(axis=1)
            assert np.all(lo >= hi)                       # top-k of every (i, p) block
        assert_array_equal(dense[kept], interp.matrix[kept])
    # nnz = 1 equals the reference global fit at keep = J*P whenever that fit is one-per-(i, p)
    sp1 = s.truncate_sparse_fixed(interp, 1)
    glob = s.truncate_sparse(interp, grid.num_points * spec.num_pairs)
    pair_g = np.searchsorted(off, glob.col_indices, side="right") - 1
    rows_g = np.repeat(np.arange(grid.num_points), np.diff(glob.row_splits))
    per = np.zeros((grid.num_points, spec.num_pairs), int)
    np.add.at(per, (rows_g, pair_g), 1)
    if np.all(per == 1):
        assert_array_equal(sp1.col_indices, glob.col_indices)


def _band(sp, off, placement=None):
    # the operator image needs a device for its upload; build the host image on CPU tensors
    from paper_2306_08514_b200 import maps
    import torch
    orig = maps.dev.device
    maps.dev.device = lambda: torch.device("cpu")
    try:
        if np.ndim(getattr(sp, "cols", np.zeros(1))) == 3:
            fx = sp
            keep = np.arange(fx.values.shape[2])[None, :] < np.asarray(fx.kept)[:, None]
            sel = np.broadcast_to(keep[:, None, :], fx.values.shape)
            rows = np.broadcast_to(np.arange(fx.values.shape[1])[None, :, None], fx.values.shape)[sel]
            return maps.BandOperator(rows, fx.cols[sel].astype(np.int64), fx.values[sel], fx.values.shape[1],
                                     int(fx.num_cols), off, placement=placement)
        j = sp.row_splits.shape[0] - 1
        rows = np.repeat(np.arange(j), np.diff(sp.row_splits))
        return maps.BandOperator(rows, sp.col_indices, sp.values, j, int(sp.num_cols), off, placement=placement)
    finally:
        maps.dev.device = orig


@pytest.mark.parametrize("permuted", [False, True])
def test_band_roundtrip_bit_exact(golden_scene, permuted):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    for tag in keep_tags(g):
        ref = sparse_from_golden(g, tag)
        groups = (grid.num_points + 3) // 4
        band = _band(ref, spec.offsets, np.arange(groups)[::-1].copy() if permuted else None)
        if permuted:   # meta bases/counts describe each slot
            assert np.array_equal(np.sort(band.group_order), np.arange(groups))
            meta = band.host_blob.reshape(-1)
            for t in range(band.tiles):
                w0 = band.host_tile_off[t] // 4
                for slot in range(8):
                    gidx = t * 8 + slot
                    if gidx < groups:
                        grp = band.group_order[gidx]
                        assert meta[w0 + 16 + slot] == 4 * grp
                        assert meta[w0 + 24 + slot] == min(4, grid.num_points - 4 * grp)
                    else:
                        assert meta[w0 + 24 + slot] == 0
        vals, cols, splits = band.to_csr()
        assert_array_equal(cols, ref.col_indices)
        assert_array_equal(splits, ref.row_splits)
        assert_array_equal(vals, ref.values.astype(np.float32))
        # every record's sample index lies inside the operator; padded weights are zero
        rtg, rs, weights, mask = band._rec
        assert np.all(rs < spec.offsets[-1]) and np.all(weights[~mask] == 0)


def test_band_empty_and_keep_all(golden_scene):
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    interp = s.build_interp_matrix(tdoa, spec, frame)
    empty = _band(s.truncate_sparse(interp, 0), spec.offsets)
    assert empty.records == 0
    full = _band(s.truncate_sparse(interp, interp.matrix.size), spec.offsets)
    groups = (grid.num_points + 3) // 4
    assert full.records == groups * spec.offsets[-1]
    assert full.max_tile_records <= 8 * int(spec.offsets[-1])


def test_errors_mirror_reference():
    assert issubclass(s.DimensionError, ValueError) and issubclass(s.DimensionError, s.SrpMapError)
    assert issubclass(s.ConfigError, ValueError)
    assert not issubclass(s.CapacityError, ValueError)
    with pytest.raises(s.InvalidGeometryError):
        s.MicrophoneArray(np.zeros((1, 3)))
    with pytest.raises(s.InvalidGridError):
        s.CandidateGrid("ff", np.array([[2.0, 0, 0]]))
    with pytest.raises(s.CapacityError):
        tdoa = s.TdoaTable(np.zeros((1000, 6)), np.ones(6))
        s.build_srp_matrix(tdoa, s.FrameSpec(512, 4000), max_bytes=10_000)
    with pytest.raises(s.ConfigError):
        s.sample_spec(s.TdoaTable(np.zeros((1, 1)), np.array([1.0])), s.FrameSpec(64, 8000))
    with pytest.raises(ValueError):
        s.FrameSpec(5, 100)


def test_partition_and_keys():
    import torch
    assert [partition(10, 3, r) for r in range(3)] == [(0, 4), (4, 3), (7, 3)]
    assert sum(partition(1000, 8, r)[1] for r in range(8)) == 1000
    # a key for value 2.5 at index 7, re-based by an offset of 100
    v = np.float32(2.5).view(np.uint32)
    hi = int(v) | 0x80000000
    key = torch.tensor([(hi << 32 | (0xFFFFFFFF - 7)) - (1 << 64)], dtype=torch.int64)
    idx, val = decode_host_keys(key)
    assert idx.item() == 7 and val.item() == 2.5
    idx, _ = decode_host_keys(offset_keys(key, 100))
    assert idx.item() == 107


def test_workloads_deterministic():
    from paper_2306_08514_b200 import workloads
    a = workloads.make("cfg1", num_frames=8)
    b = workloads.make("cfg1", num_frames=8)
    assert_array_equal(a.samples, b.samples)
    assert a.grid.num_points == 1681 and a.pairs.num_pairs == 6
    assert a.samples.shape == (4, 7 * 512 + 1024)


def test_fixed_nnz_from_tdoa_matches_dense_fit(golden_scene):
    """The cfg4-scale builder (no dense Lambda) equals the dense per-(i, p) top-k fit bit for bit."""
    from paper_2306_08514_b200.operators import sparse_interp_fixed
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    interp = s.build_interp_matrix(tdoa, spec, frame)
    for nnz in (1, 2, 3, 8):
        a = s.truncate_sparse_fixed(interp, nnz)
        fx = sparse_interp_fixed(tdoa, spec, frame, nnz)
        b = fx.to_csr()
        assert_array_equal(a.col_indices, b.col_indices)
        assert_array_equal(a.row_splits, b.row_splits)
        assert_array_equal(a.values, b.values)
        assert fx.num_kept == a.num_kept
        vals, cols, splits = _band(fx, spec.offsets).to_csr()
        assert_array_equal(cols, a.col_indices)
        assert_array_equal(splits, a.row_splits)
        assert_array_equal(vals, a.values.astype(np.float32))


def test_streamed_global_fit_matches_reference(golden_scene):
    """truncate_sparse_streamed (row-blocked, two-pass histogram selection, never the dense
    operator) reproduces the reference's global top-Q CSR bit for bit (interpolation.py:155-175)."""
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    for tag in keep_tags(g):
        ref = sparse_from_golden(g, tag)
        got = s.truncate_sparse_streamed(tdoa, spec, frame, int(ref.values.shape[0]), block_bytes=1 << 14)
        assert np.array_equal(got.col_indices, ref.col_indices)
        assert np.array_equal(got.row_splits, ref.row_splits)
        assert np.array_equal(got.values, ref.values)
    with pytest.raises(ValueError):
        s.truncate_sparse_streamed(tdoa, spec, frame, -1)


def _nonzero_rows(splits, cols, vals):
    """Per row: the (column, float32 weight) entries whose weight is not 0, in CSR order."""
    out = []
    for i in range(splits.shape[0] - 1):
        a, b = int(splits[i]), int(splits[i + 1])
        v = np.asarray(vals[a:b], dtype=np.float32)
        keep = v != 0
        out.append((np.asarray(cols[a:b])[keep].astype(np.int64), v[keep]))
    return out


def test_sell_layout_decodes_to_reference_csr(golden_scene):
    """The fused chain's sliced-ELL image holds exactly the reference CSR (interpolation.py:
    155-175): candidate i's k-th entry sits at row chunk_off[i // 32] + k, lane i % 32, with
    the reference column and float32(value); every other slot is padding of weight 0."""
    _, g = golden_scene
    for tag in keep_tags(g):
        sp = sparse_from_golden(g, tag)
        c, v, off = s.maps.sell_layout(sp)
        splits = np.asarray(sp.row_splits)
        nnz = np.diff(splits)
        j = nnz.shape[0]
        used = np.zeros(v.shape, dtype=bool)
        for i in range(j):
            r0, lane = int(off[i // 32]), i % 32
            k = int(nnz[i])
            assert_array_equal(c[r0:r0 + k, lane].astype(np.int64), sp.col_indices[splits[i]:splits[i + 1]])
            assert_array_equal(v[r0:r0 + k, lane], np.asarray(sp.values[splits[i]:splits[i + 1]], np.float32))
            used[r0:r0 + k, lane] = True
        assert np.all(v[~used] == 0)                       # padding never contributes
        w = np.diff(off)
        assert np.all(w >= np.pad(nnz, (0, (-j) % 32)).reshape(-1, 32).max(axis=1))


@pytest.mark.parametrize("mode", ["compact", "runs", "contiguous"])
@pytest.mark.parametrize("group", [4, 8])
def test_tile_layout_holds_the_csr(golden_scene, group, mode):
    """The gathered-window image (tiles.TileLayout, 4-lag groups for the 3xTF32 kernel, 8 for
    fp16 / bf16; compact bisected tiles, tiles of aligned 8-candidate runs, tiles of 256
    consecutive candidates): every candidate sits in exactly one tile row, and decoding the
    slabs (tile row, group_col + lag offset, natural -> storage column) gives exactly the
    CSR's nonzero entries with float32 weights; the remaining slab entries are 0."""
    from paper_2306_08514_b200 import tiles
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    off = s.sampling.spec_offsets(spec)
    perm = tiles.natural_columns(off)                      # natural index -> storage column
    for tag in keep_tags(g):
        sp = sparse_from_golden(g, tag)
        j = int(np.asarray(sp.row_splits).shape[0] - 1)
        lay = tiles.TileLayout(sp, off, j, group=group, runs=(mode == "runs"), contiguous=(mode == "contiguous"))
        if mode == "contiguous":
            assert_array_equal(lay.tile_rows.ravel()[:j], np.arange(j))
        if mode == "runs":       # whole aligned runs of 8 candidates, in ascending tile rows
            first = lay.tile_rows[:, ::8]
            assert np.all(first[first >= 0] % 8 == 0)
        # the valid rows of a tile are a prefix (the kernel's epilogue counts on it)
        valid = lay.tile_rows >= 0
        assert np.all(valid[:, :-1] >= valid[:, 1:])
        rows_used = lay.tile_rows[lay.tile_rows >= 0]
        assert_array_equal(np.sort(rows_used), np.arange(j))
        assert_array_equal(lay.tile_pos[lay.tile_rows[lay.tile_rows >= 0]], np.flatnonzero(lay.tile_rows.ravel() >= 0))
        per = tiles.SLAB // group
        got = [dict() for _ in range(j)]
        for t in range(lay.num_tiles):
            b0, nk = int(lay.tile_slab[t]), int(lay.tile_nkb[t])
            cols = (lay.group_col[b0 * per:(b0 + nk) * per][:, None] + np.arange(group)[None, :]).ravel()
            for h in range(2):
                a = lay.slabs[2 * b0 + h:2 * (b0 + nk):2].transpose(1, 0, 2).reshape(tiles.HALF, nk * tiles.SLAB)
                for r in range(tiles.HALF):
                    cand = int(lay.tile_rows[t, h * tiles.HALF + r])
                    nzk = np.flatnonzero(a[r])
                    if cand < 0:
                        assert nzk.size == 0
                        continue
                    for k in nzk:
                        col = int(perm[cols[k]])
                        assert col not in got[cand]
                        got[cand][col] = a[r, k]
        ref = _nonzero_rows(np.asarray(sp.row_splits), np.asarray(sp.col_indices), np.asarray(sp.values))
        for i in range(j):
            rc, rv = ref[i]
            assert sorted(got[i]) == sorted(rc.tolist())
            assert all(got[i][int(cc)] == vv for cc, vv in zip(rc, rv))


def test_candidate_blocks_are_row_slices(golden_scene):
    """candidate_block (the candidate partition's per-rank operator) keeps exactly the
    operator's rows [first, first + count): CSR rows, fixed-nnz rows, TDOA rows."""
    from paper_2306_08514_b200 import distributed as D
    _, g = golden_scene
    array, pairs, grid, frame, tdoa, spec = scene_objects(g)
    sp = sparse_from_golden(g, keep_tags(g)[0])
    j = int(np.asarray(sp.row_splits).shape[0] - 1)
    parts = [D.partition(j, 3, r) for r in range(3)]
    blocks = [D.candidate_block(sp, a, n) for a, n in parts]
    assert sum(b.num_rows for b in blocks) == j
    dense = np.zeros((j, sp.num_cols))
    dense[np.repeat(np.arange(j), np.diff(sp.row_splits)), sp.col_indices] = sp.values
    for (a, n), b in zip(parts, blocks):
        d = np.zeros((n, sp.num_cols))
        d[np.repeat(np.arange(n), np.diff(b.row_splits)), b.col_indices] = b.values
        assert_array_equal(d, dense[a:a + n])
    fx = s.sparse_interp_fixed(tdoa, spec, frame, 2)
    fb = D.candidate_block(fx, parts[1][0], parts[1][1])
    assert_array_equal(fb.values, fx.values[:, parts[1][0]:parts[1][0] + parts[1][1]])
    st = D.candidate_block(s.steering_operator(tdoa, frame), parts[2][0], parts[2][1])
    assert_array_equal(st.tdoa.delta_t, tdoa.delta_t[parts[2][0]:])
    assert st.num_candidates == parts[2][1]
