"""Host-side operator construction (precomputed once, then uploaded).

Same operators and semantics as the reference builders:
  SrpMatrix / build_srp_matrix          srp.py:22-62
  LowRankSrp / truncate_srp_matrix      lowrank.py:19-48
  InterpMatrix / build_interp_matrix    interpolation.py:27-44, 93-105
  LowRankInterp / truncate_low_rank     interpolation.py:47-65, 139-152
  SparseInterp / truncate_sparse        interpolation.py:68-90, 155-175
plus `truncate_sparse_fixed`, the fixed-nnz-per-(candidate, pair) fit used by
the BASELINE nnz sweep (its map is still the reference `sspi_map` applied to
the resulting CSR).  These stay float64 NumPy: they are fitted once per scene
and are not on the per-frame device path.
"""

from __future__ import annotations

from dataclasses import dataclass

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .errors import CapacityError, DimensionError

DEFAULT_MATRIX_CAP_BYTES = 2 * 1024 ** 3


def check_capacity(shape, itemsize: int, max_bytes: int, what: str) -> None:
    need = shape[0] * shape[1] * itemsize
    if need > max_bytes:
        raise CapacityError(f"{what} of shape {shape} needs {need / 1e9:.2f} GB, above the cap "
                            f"of {max_bytes / 1e9:.2f} GB")


# ---------------------------------------------------------------- conventional

@dataclass(frozen=True)
class SrpMatrix:
    matrix: np.ndarray   # (J, P*B) complex
    num_pairs: int
    num_bins: int

    @property
    def num_candidates(self) -> int:
        return self.matrix.shape[0]

    def pair_block(self, p: int) -> np.ndarray:
        return self.matrix[:, p * self.num_bins:(p + 1) * self.num_bins]


def srp_matrix_shape(tdoa, frame):
    return tdoa.num_candidates, tdoa.num_pairs * frame.num_bins


def build_srp_matrix(tdoa, frame, max_bytes: int = DEFAULT_MATRIX_CAP_BYTES) -> SrpMatrix:
    """H[i, p B + k - 1] = exp(j w_k dt_p(i))."""
    shape = srp_matrix_shape(tdoa, frame)
    check_capacity(shape, 16, max_bytes, "SRP matrix")
    b = frame.num_bins
    w = frame.bin_freqs
    out = np.empty(shape, dtype=np.complex128)
    for p in range(tdoa.num_pairs):
        np.exp(1j * tdoa.delta_t[:, p:p + 1] * w[None, :], out=out[:, p * b:(p + 1) * b])
    return SrpMatrix(matrix=out, num_pairs=tdoa.num_pairs, num_bins=b)


@dataclass(frozen=True)
class LowRankSrp:
    tall: np.ndarray            # (J, R) complex = U[:, :R] s[:R]
    fat: np.ndarray             # (R, P*B) complex = Vh[:R]
    singular_values: np.ndarray

    @property
    def rank(self) -> int:
        return self.tall.shape[1]

    def to_dense(self) -> np.ndarray:
        return self.tall @ self.fat


def low_rank_srp_from_svd(u, s, vt, rank: int) -> LowRankSrp:
    return LowRankSrp(tall=u[:, :rank] * s[:rank], fat=vt[:rank], singular_values=s[:rank].copy())


def truncate_srp_matrix(srp, rank: int) -> LowRankSrp:
    full = min(srp.matrix.shape)
    if not 1 <= rank <= full:
        raise ValueError(f"rank must be in [1, {full}], got {rank}")
    u, s, vt = np.linalg.svd(srp.matrix, full_matrices=False)
    return low_rank_srp_from_svd(u, s, vt, rank)


# ---------------------------------------------------------------- interpolation

@dataclass(frozen=True)
class InterpMatrix:
    matrix: np.ndarray   # (J, S) float64
    spec: object

    @property
    def num_candidates(self) -> int:
        return self.matrix.shape[0]

    @property
    def num_samples(self) -> int:
        return self.matrix.shape[1]

    def pair_block(self, p: int) -> np.ndarray:
        off = _offsets(self.spec)
        return self.matrix[:, off[p]:off[p + 1]]


def _offsets(spec) -> np.ndarray:
    counts = np.asarray(spec.counts, dtype=np.int64)
    return np.concatenate([[0], np.cumsum(2 * counts + 1)]).astype(np.int64)


def _lags(count: int) -> np.ndarray:
    return np.concatenate([np.arange(count + 1), np.arange(-count, 0)])


def build_interp_matrix(tdoa, spec, frame, max_bytes: int = DEFAULT_MATRIX_CAP_BYTES) -> InterpMatrix:
    """Lambda[:, off_p + s] = sinc(dt_p(i)/T - lag_s) (normalized sinc)."""
    if tdoa.num_pairs != spec.num_pairs:
        raise DimensionError("TDOA table and sample spec disagree on pair count")
    off = _offsets(spec)
    shape = (tdoa.num_candidates, int(off[-1]))
    check_capacity(shape, 8, max_bytes, "interpolation matrix")
    out = np.empty(shape)
    for p in range(spec.num_pairs):
        frac = tdoa.delta_t[:, p] / frame.sample_period
        out[:, off[p]:off[p + 1]] = np.sinc(frac[:, None] - _lags(int(spec.counts[p]))[None, :])
    return InterpMatrix(matrix=out, spec=spec)


@dataclass(frozen=True)
class LowRankInterp:
    tall: np.ndarray            # (J, R)
    fat: np.ndarray             # (R, S)
    singular_values: np.ndarray

    @property
    def rank(self) -> int:
        return self.tall.shape[1]

    def to_dense(self) -> np.ndarray:
        return self.tall @ self.fat


def low_rank_interp_from_svd(u, s, vt, rank: int) -> LowRankInterp:
    return LowRankInterp(tall=u[:, :rank] * s[:rank], fat=vt[:rank], singular_values=s[:rank].copy())


def truncate_low_rank(interp, rank: int) -> LowRankInterp:
    full = min(interp.matrix.shape)
    if not 1 <= rank <= full:
        raise ValueError(f"rank must be in [1, {full}], got {rank}")
    u, s, vt = np.linalg.svd(interp.matrix, full_matrices=False)
    return low_rank_interp_from_svd(u, s, vt, rank)


@dataclass(frozen=True)
class SparseInterp:
    values: np.ndarray        # (Q,)
    col_indices: np.ndarray   # (Q,) int64
    row_splits: np.ndarray    # (J+1,) int64
    num_cols: int

    @property
    def num_rows(self) -> int:
        return self.row_splits.shape[0] - 1

    @property
    def num_kept(self) -> int:
        return self.values.shape[0]

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.num_rows, self.num_cols))
        rows = np.repeat(np.arange(self.num_rows), np.diff(self.row_splits))
        out[rows, self.col_indices] = self.values
        return out


def _csr_from_flat(mat: np.ndarray, sel: np.ndarray) -> SparseInterp:
    sel = np.sort(sel)
    rows = sel // mat.shape[1]
    cols = sel % mat.shape[1]
    splits = np.zeros(mat.shape[0] + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=mat.shape[0]), out=splits[1:])
    return SparseInterp(values=mat.ravel()[sel], col_indices=cols.astype(np.int64),
                        row_splits=splits, num_cols=mat.shape[1])


def truncate_sparse(interp, keep: int) -> SparseInterp:
    """Global top-`keep` magnitudes; ties go to the lower row-major flat index.

    Same selection as the reference's stable argsort of -|Lambda|
    (interpolation.py:166-170), computed by thresholding: everything strictly
    above the keep-th largest magnitude, then the first ties in flat order.
    """
    mat = interp.matrix
    size = mat.size
    if not 0 <= keep <= size:
        raise ValueError(f"keep must be in [0, {size}], got {keep}")
    mag = np.abs(mat).ravel()
    if keep == 0:
        sel = np.zeros(0, dtype=np.int64)
    elif keep == size:
        sel = np.arange(size, dtype=np.int64)
    else:
        thresh = np.partition(mag, size - keep)[size - keep]
        above = np.flatnonzero(mag > thresh)
        ties = np.flatnonzero(mag == thresh)[:keep - above.size]
        sel = np.concatenate([above, ties])
    return _csr_from_flat(mat, sel)


def interp_rows(tdoa, spec, frame, r0: int, r1: int) -> np.ndarray:
    """Rows r0..r1-1 of build_interp_matrix, element for element the same float64 values
    (the same per-element expression on a row slice of the TDOA table)."""
    off = _offsets(spec)
    out = np.empty((r1 - r0, int(off[-1])))
    for p in range(spec.num_pairs):
        frac = tdoa.delta_t[r0:r1, p] / frame.sample_period
        out[:, off[p]:off[p + 1]] = np.sinc(frac[:, None] - _lags(int(spec.counts[p]))[None, :])
    return out


_HIST_SHIFT = 44     # histogram bin = top 20 bits of the float64 magnitude (exponent + 8 mantissa bits)


def truncate_sparse_streamed(tdoa, spec, frame, keep: int, block_bytes: int = 1 << 28) -> SparseInterp:
    """`truncate_sparse(build_interp_matrix(tdoa, spec, frame), keep)` -- the reference's
    global top-`keep` rule (interpolation.py:155-175: stable argsort of -|Lambda|, ties to
    the lower row-major flat index) -- without ever holding the dense J x S operator
    (18.7 GB at BASELINE cfg4; the reference's argsort would also need its int64 index
    array and scratch).  Two streamed passes over row blocks:

    1. histogram of the magnitudes' float64 bit patterns (monotone for |x| >= 0) on their
       top 20 bits -> the bin b* holding the keep-th largest magnitude;
    2. every entry in a bin above b* is kept; the entries of bin b* are ranked by
       (-|value|, flat index) and the first keep - (count above) are kept.

    The values are recomputed per block exactly as build_interp_matrix computes them, so
    the selection and the CSR are bit-identical to truncate_sparse on the dense matrix.
    """
    off = _offsets(spec)
    j, s = tdoa.num_candidates, int(off[-1])
    size = j * s
    if not 0 <= keep <= size:
        raise ValueError(f"keep must be in [0, {size}], got {keep}")
    rows_per = max(1, int(block_bytes // (8 * max(s, 1))))
    blocks = [(r0, min(j, r0 + rows_per)) for r0 in range(0, j, rows_per)]

    def magnitude_bins(block):
        mag = np.abs(block).ravel()
        return mag, (mag.view(np.uint64) >> np.uint64(_HIST_SHIFT)).astype(np.int64)

    if keep == 0 or keep == size:
        sel_rows, sel_cols, sel_vals = [], [], []
        for r0, r1 in blocks:
            blk = interp_rows(tdoa, spec, frame, r0, r1) if keep else np.zeros((0, s))
            if keep:
                sel_rows.append(np.repeat(np.arange(r0, r1), s))
                sel_cols.append(np.tile(np.arange(s), r1 - r0))
                sel_vals.append(blk.ravel())
        return _csr_from_parts(sel_rows, sel_cols, sel_vals, j, s)
    nbins = 1 << (64 - _HIST_SHIFT)

    def pass1(blk_range):
        _, bins = magnitude_bins(interp_rows(tdoa, spec, frame, *blk_range))
        return np.bincount(bins, minlength=nbins)

    def pass2(blk_range):
        r0, r1 = blk_range
        blk = interp_rows(tdoa, spec, frame, r0, r1)
        _, bins = magnitude_bins(blk)
        flat = blk.ravel()
        hi = np.flatnonzero(bins > b_star)
        mid = np.flatnonzero(bins == b_star)
        return r0 + hi // s, hi % s, flat[hi], r0 * s + mid, flat[mid]

    # blocks run on host threads (the NumPy kernels release the GIL); results are combined
    # in block order, so the output does not depend on the thread count
    workers = max(1, min(len(blocks), os.cpu_count() or 1))
    with ThreadPoolExecutor(max_workers=workers) as pool:
        hist = np.zeros(nbins, dtype=np.int64)
        for h in pool.map(pass1, blocks):
            hist += h
        from_top = np.cumsum(hist[::-1])[::-1]           # count of entries in bins >= b
        b_star = int(np.flatnonzero(from_top >= keep)[-1])
        above = int(from_top[b_star + 1]) if b_star + 1 < nbins else 0
        need = keep - above
        parts = list(pool.map(pass2, blocks))
    rows_k, cols_k, vals_k = [p[0] for p in parts], [p[1] for p in parts], [p[2] for p in parts]
    tf, tv = np.concatenate([p[3] for p in parts]), np.concatenate([p[4] for p in parts])
    order = np.lexsort((tf, -np.abs(tv)))[:need]          # primary -|v|, then flat index
    rows_k.append(tf[order] // s)
    cols_k.append(tf[order] % s)
    vals_k.append(tv[order])
    return _csr_from_parts(rows_k, cols_k, vals_k, j, s)


def _csr_from_parts(rows, cols, vals, num_rows: int, num_cols: int) -> SparseInterp:
    r = np.concatenate(rows).astype(np.int64) if rows else np.zeros(0, dtype=np.int64)
    c = np.concatenate(cols).astype(np.int64) if cols else np.zeros(0, dtype=np.int64)
    v = np.concatenate(vals) if vals else np.zeros(0)
    order = np.argsort(r * num_cols + c, kind="stable")
    splits = np.zeros(num_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=num_rows), out=splits[1:])
    return SparseInterp(values=v[order], col_indices=c[order], row_splits=splits, num_cols=num_cols)


def truncate_sparse_fixed(interp, nnz: int) -> SparseInterp:
    """Keep the `nnz` largest |entries| of every (candidate, pair) block.

    Ties go to the lower column (stable).  Blocks narrower than nnz are kept
    whole, so Q = sum_p min(nnz, 2 N_p + 1) * J.  This is the fixed-width
    ELL fit of the BASELINE nnz sweep; at nnz = 1 it coincides with the
    reference's global fit at keep = J*P whenever that fit keeps exactly one
    entry per (candidate, pair).
    """
    if nnz < 0:
        raise ValueError("nnz must be >= 0")
    mat = interp.matrix
    off = _offsets(interp.spec)
    j = mat.shape[0]
    picks = []
    for p in range(len(off) - 1):
        block = np.abs(mat[:, off[p]:off[p + 1]])
        k = min(nnz, block.shape[1])
        if k == 0:
            continue
        idx = np.argsort(-block, axis=1, kind="stable")[:, :k] + off[p]
        picks.append((np.arange(j)[:, None] * mat.shape[1] + idx).ravel())
    sel = np.concatenate(picks) if picks else np.zeros(0, dtype=np.int64)
    return _csr_from_flat(mat, sel)


def resolve_sparsity(token, num_candidates: int, num_pairs: int, size: int) -> int:
    """"all" | "<x>jp" | int -> kept count (config.py:245-262)."""
    if token == "all":
        return size
    if isinstance(token, str) and token.endswith("jp"):
        return int(round(float(token[:-2]) * num_candidates * num_pairs))
    return int(token)


@dataclass(frozen=True)
class FixedNnzInterp:
    """Fixed-nnz-per-(candidate, pair) sparse interpolation operator, pair-blocked.

    cols[p, i, :] are absolute sample indices (ascending), values[p, i, :] the
    float64 sinc weights; every (candidate, pair) keeps min(nnz, 2 N_p + 1)
    entries (shorter pair blocks are padded with value 0 at their first column).
    It is exactly `truncate_sparse_fixed(build_interp_matrix(...), nnz)` but is
    built pair by pair from the TDOA table, so the dense J x S operator (18.7 GB at
    BASELINE cfg4) never exists.  `to_csr()` gives the reference `SparseInterp`.
    """

    values: np.ndarray      # (P, J, k) float64
    cols: np.ndarray        # (P, J, k) int32
    kept: np.ndarray        # (P,) entries really kept per (i, p)
    num_cols: int

    @property
    def num_rows(self) -> int:
        return self.values.shape[1]

    @property
    def num_kept(self) -> int:
        return int(np.sum(self.kept)) * self.num_rows

    def to_csr(self) -> SparseInterp:
        p_count, j, _ = self.values.shape
        rows, cols, vals = [], [], []
        for p in range(p_count):
            k = int(self.kept[p])
            rows.append(np.repeat(np.arange(j), k))
            cols.append(self.cols[p, :, :k].ravel().astype(np.int64))
            vals.append(self.values[p, :, :k].ravel())
        r, c, v = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
        order = np.lexsort((c, r))
        splits = np.zeros(j + 1, dtype=np.int64)
        np.cumsum(np.bincount(r, minlength=j), out=splits[1:])
        return SparseInterp(values=v[order], col_indices=c[order], row_splits=splits,
                            num_cols=self.num_cols)


def sparse_interp_fixed(tdoa, spec, frame, nnz: int, rows=None) -> FixedNnzInterp:
    """Per (candidate, pair): the `nnz` largest |sinc(dt fs - n)|, ties to the lower column.

    |sinc(x - n)| = |sin(pi x)| / (pi |x - n|) decreases with |x - n|, so the winners
    lie among the nnz + 2 lags nearest to x; those are evaluated exactly as
    build_interp_matrix does (np.sinc on float64) and ranked by a stable sort on
    (-|value|, column), which reproduces the full-block argsort of
    truncate_sparse_fixed.  `rows` optionally restricts to a candidate subset.
    """
    if nnz < 1:
        raise ValueError("nnz must be >= 1")
    off = _offsets(spec)
    delta = tdoa.delta_t if rows is None else tdoa.delta_t[rows]
    j, p_count = delta.shape
    kmax = int(min(nnz, np.max(2 * np.asarray(spec.counts) + 1)))
    values = np.zeros((p_count, j, kmax))
    cols = np.zeros((p_count, j, kmax), dtype=np.int32)
    kept = np.zeros(p_count, dtype=np.int64)
    for p in range(p_count):
        c = int(spec.counts[p])
        width = 2 * c + 1
        k = min(nnz, width)
        kept[p] = k
        cols[p, :, :] = off[p]
        x = delta[:, p] / frame.sample_period
        span = min(width, k + 2)
        base = np.floor(x).astype(np.int64) - (span - 1) // 2
        base = np.clip(base, -c, c - span + 1)
        lags = base[:, None] + np.arange(span)[None, :]                 # signed lags, ascending
        vals = np.sinc(x[:, None] - lags)
        colid = np.where(lags >= 0, lags, width + lags)                  # storage order 0..N, -N..-1
        # stable ranking per row: primary -|v|, secondary column id
        key = np.argsort(colid, axis=1, kind="stable")
        v_s = np.take_along_axis(vals, key, 1)
        c_s = np.take_along_axis(colid, key, 1)
        rank = np.argsort(-np.abs(v_s), axis=1, kind="stable")[:, :k]
        sel_c = np.take_along_axis(c_s, rank, 1)
        sel_v = np.take_along_axis(v_s, rank, 1)
        # near-integer x: the off-peak sinc values are rounding noise (sin(pi n) != 0 in
        # floating point) and not monotone in |x - n|; rank those rows over the whole block
        odd = np.flatnonzero(np.min(np.abs(sel_v), axis=1) < 1e-9) if k > 1 else np.zeros(0, int)
        if odd.size:
            full = np.sinc(x[odd, None] - _lags(c)[None, :])          # storage order
            r2 = np.argsort(-np.abs(full), axis=1, kind="stable")[:, :k]
            sel_c[odd] = r2
            sel_v[odd] = np.take_along_axis(full, r2, 1)
        back = np.argsort(sel_c, axis=1, kind="stable")
        cols[p, :, :k] = np.take_along_axis(sel_c, back, 1) + off[p]
        values[p, :, :k] = np.take_along_axis(sel_v, back, 1)
    return FixedNnzInterp(values=values, cols=cols, kept=kept, num_cols=int(off[-1]))


@dataclass(frozen=True)
class SteeringTdoa:
    """The conventional operator H[i, pB+k-1] = exp(j w_k dt_p(i)) kept implicit.

    `srp_map_exact` accepts it wherever it accepts an `SrpMatrix` (srp.py:22-62): the
    GPU generates H on chip from the TDOA table instead of reading it from memory, so
    grids whose H cannot be stored (BASELINE cfg4: 334611 x 61320 complex) still map.
    """

    tdoa: object
    frame: object

    @property
    def num_pairs(self) -> int:
        return self.tdoa.num_pairs

    @property
    def num_bins(self) -> int:
        return self.frame.num_bins

    @property
    def num_candidates(self) -> int:
        return self.tdoa.num_candidates

    def materialize(self, max_bytes: int = DEFAULT_MATRIX_CAP_BYTES) -> SrpMatrix:
        return build_srp_matrix(self.tdoa, self.frame, max_bytes)


def steering_operator(tdoa, frame) -> SteeringTdoa:
    return SteeringTdoa(tdoa=tdoa, frame=frame)
