"""SRP map backends on the GPU: conventional, LR, SI, SLRI, SSPI, and argmax.

Drop-ins for srp.srp_map_exact (srp.py:65-71), srp.locate (:74-80),
lowrank.lr_map (lowrank.py:51-57), interpolation.si_map / slri_map / sspi_map
(interpolation.py:129-136, 178-195) and cli.evaluate_map (cli.py:170-180).
Same arguments and DimensionError checks; inputs may carry a leading frame
axis; maps are returned as device tensors (J,) or (F, J) float32.

Every map function also takes keyword-only `argmax=True` to return
(z, index) with the per-frame argmax fused into the map kernel (index int64,
ties to the lowest candidate index), and `out_map=False` to skip writing z
(argmax-only output).

Operators are converted to device layouts once per operator object
(`_device.CACHE`): the SSPI operator becomes a tiled-band record array, low-rank
factors are cast to float32 (complex factors folded into real ones), and the
steering matrix is stored as interleaved (Re H, -Im H) rows for the
tensor-core GEMM.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _device as dev
from . import _native as nat
from . import tiles
from .errors import DimensionError
from .sampling import TdGccSamples, spec_offsets


# ----------------------------------------------------------------- helpers

def _new_keys(frames: int, want: bool, num_candidates: int | None = None):
    if not want:
        return None
    if num_candidates == 0:     # np.argmax of an empty map raises (srp.py:74-80)
        raise ValueError("attempt to get argmax of an empty sequence (the map has no candidates)")
    return torch.empty(frames, dtype=torch.int64, device=dev.device())


def decode_keys(keys: torch.Tensor):
    """Packed argmax keys -> (index int64, value float32) device tensors."""
    idx = torch.empty(keys.shape[0], dtype=torch.int64, device=keys.device)
    val = torch.empty(keys.shape[0], dtype=torch.float32, device=keys.device)
    nat.call("srpgpu_decode_keys", dev.ptr(keys), keys.shape[0], dev.ptr(idx), dev.ptr(val),
             dev.stream_ptr())
    return idx, val


def _finish(z, keys, batched: bool, argmax: bool):
    zz = None if z is None else (z if batched else z[0])
    if not argmax:
        return zz
    idx, _ = decode_keys(keys)
    return zz, (idx if batched else idx[0])


def _gcc_matrix(gcc, num_pairs: int, num_bins: int):
    """(F, P*B) complex64 device tensor + batched flag, with the reference shape check."""
    vals = gcc if isinstance(gcc, (torch.Tensor, np.ndarray)) else gcc.values
    v = dev.as_c64(vals)
    batched = v.dim() == 2
    if v.shape[-1] != num_pairs * num_bins:
        raise DimensionError(f"cross-spectrum of shape {tuple(v.shape)} does not match "
                             f"{num_pairs} pairs x {num_bins} bins")
    return v.reshape(-1, num_pairs * num_bins), batched


def _sample_matrix(samples, num_cols: int):
    vals = samples.values if (not isinstance(samples, (torch.Tensor, np.ndarray, list, tuple))
                               and hasattr(samples, "spec")) else samples
    x = dev.as_f32(vals)
    batched = x.dim() == 2
    if x.shape[-1] != num_cols or x.dim() > 2:
        raise DimensionError(f"sample vector of shape {tuple(x.shape)} does not match operator "
                             f"with {num_cols} columns")
    return x.reshape(-1, num_cols), batched


def _lag_major(samples, num_cols: int):
    """(buf (S, ld) lag-major f32, frames, batched) for any samples input.

    Kernel-produced TdGccSamples already carry the lag-major buffer; anything else
    (reference TdGccSamples, arrays, tensors) is transposed on the device once.
    """
    buf = getattr(samples, "lag_major", None)
    if buf is not None and buf.shape[0] == num_cols:
        vals = samples.values
        batched = vals.dim() == 2
        return buf, (vals.shape[0] if batched else 1), batched
    x, batched = _sample_matrix(samples, num_cols)
    f = x.shape[0]
    ld = (f + 3) // 4 * 4
    buf = torch.empty((num_cols, ld), dtype=torch.float32, device=x.device)
    nat.call("srpgpu_transpose", dev.ptr(x), f, num_cols, num_cols, dev.ptr(buf), ld, dev.stream_ptr())
    return buf, f, batched


def _sample_offsets(samples, num_cols: int) -> np.ndarray:
    spec = getattr(samples, "spec", None)
    if spec is not None:
        off = spec_offsets(spec)
        if int(off[-1]) == num_cols:
            return off
    return np.array([0, num_cols], dtype=np.int64)   # no pair structure: one block


# ----------------------------------------------------------------- SSPI / SI

class BandOperator:
    """Tiled band image of a sparse interpolation operator (what the SSPI kernel reads).

    Candidates are cut into groups of 4 consecutive rows; groups are placed 8 to a
    tile.  For each (group, pair) the union of the sample indices kept by the group's
    candidates becomes records {u32 sample index, 3 pad, f32 weight[4]}.  Tile blob =
    meta[32] u32 (start record of slots 0..7, the record total, 7 spare; first
    candidate of slots 0..7; candidates in slots 0..7; 128 bytes) + records,
    slot-major (then pair, then ascending sample index); `tile_off` holds the blob
    byte offsets.

    Groups are placed in index order unless `placement` (a permutation of the
    groups) says otherwise; a candidate's accumulation order does not depend on its
    placement, so the maps are bit-identical either way.  (Lag-space locality
    orderings were measured at cfg3/cfg4 and gave no gain, so none is applied.)
    `mask` (host) marks the (record, candidate) slots that are real kept entries, so
    the image decodes back to the reference CSR exactly (`to_csr`).
    """

    TILE, GROUP, META_WORDS = 32, 4, 32

    def __init__(self, rows, cols, vals, num_rows: int, num_cols: int, offsets: np.ndarray,
                 placement=None):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        p_count = offsets.shape[0] - 1
        ngrp = self.TILE // self.GROUP
        groups = max(1, (num_rows + self.GROUP - 1) // self.GROUP)
        tiles = (groups + ngrp - 1) // ngrp
        pair = np.searchsorted(offsets, cols, side="right") - 1
        grp = rows // self.GROUP
        c = rows % self.GROUP
        order = np.arange(groups, dtype=np.int64) if placement is None else \
            np.asarray(placement, dtype=np.int64)
        if order.shape != (groups,) or not np.array_equal(np.sort(order), np.arange(groups)):
            raise ValueError("placement must be a permutation of the candidate groups")
        slot_of = np.empty(groups, dtype=np.int64)
        slot_of[order] = np.arange(groups, dtype=np.int64)        # group -> tile * 8 + slot
        key = (slot_of[grp] * p_count + pair) * num_cols + cols
        uniq, inv = np.unique(key, return_inverse=True)
        nrec = uniq.shape[0]
        rs = uniq % num_cols
        rtg = uniq // num_cols // p_count                 # tile * 8 + slot
        weights = np.zeros((nrec, self.GROUP), dtype=np.float32)
        mask = np.zeros((nrec, self.GROUP), dtype=bool)
        weights[inv, c] = vals.astype(np.float32)
        mask[inv, c] = True
        counts = np.bincount(rtg, minlength=tiles * ngrp).reshape(tiles, ngrp)
        tile_recs = counts.sum(axis=1)
        words = self.META_WORDS + 8 * tile_recs           # u32 words per tile blob
        tile_off_w = np.concatenate([[0], np.cumsum(words)]).astype(np.int64)
        blob = np.zeros(int(tile_off_w[-1]), dtype=np.uint32)
        starts = np.cumsum(counts, axis=1) - counts
        meta_idx = tile_off_w[:-1, None] + np.arange(ngrp)[None, :]
        blob[meta_idx.ravel()] = starts.astype(np.uint32).ravel()
        blob[tile_off_w[:-1] + ngrp] = tile_recs.astype(np.uint32)
        placed = np.full(tiles * ngrp, -1, dtype=np.int64)
        placed[:groups] = order                           # slot -> group (-1: empty slot)
        first = np.where(placed >= 0, placed * self.GROUP, 0)
        ncand = np.where(placed >= 0, np.clip(num_rows - placed * self.GROUP, 0, self.GROUP), 0)
        blob[(meta_idx + 16).ravel()] = first.astype(np.uint32)
        blob[(meta_idx + 24).ravel()] = ncand.astype(np.uint32)
        rec_tile = rtg // ngrp
        first_rec = np.concatenate([[0], np.cumsum(tile_recs)])[:-1]
        local = np.arange(nrec) - first_rec[rec_tile]
        base = tile_off_w[rec_tile] + self.META_WORDS + 8 * local
        blob[base] = rs.astype(np.uint32)
        for k in range(self.GROUP):
            blob[base + 4 + k] = weights[:, k].view(np.uint32)
        self.num_rows, self.num_cols, self.num_pairs = num_rows, num_cols, p_count
        self.offsets = offsets
        self.records = nrec
        self.tiles = tiles
        self.max_tile_records = int(tile_recs.max()) if tile_recs.size else 0
        self.max_pair_records = self.max_tile_records
        self.host_blob = blob
        self.host_tile_off = tile_off_w * 4
        self.group_order = order
        self._rec = (placed[rtg], rs, weights, mask)
        self.d_blob = torch.from_numpy(blob.view(np.int32)).to(dev.device()) if blob.size else \
            torch.zeros(16, dtype=torch.int32, device=dev.device())
        self.d_tile_off = dev.as_i64(self.host_tile_off)

    @classmethod
    def from_csr(cls, values, cols, splits, num_cols: int, offsets):
        splits = np.asarray(splits, dtype=np.int64)
        j = splits.shape[0] - 1
        rows = np.repeat(np.arange(j, dtype=np.int64), np.diff(splits))
        return cls(rows, cols, values, j, num_cols, offsets)

    @classmethod
    def from_fixed(cls, fx, offsets):
        p_count, j, k = fx.values.shape
        keep = np.arange(k)[None, :] < np.asarray(fx.kept)[:, None]          # (P, k)
        sel = np.broadcast_to(keep[:, None, :], fx.values.shape)
        rows = np.broadcast_to(np.arange(j, dtype=np.int64)[None, :, None], fx.values.shape)[sel]
        return cls(rows, fx.cols[sel].astype(np.int64), fx.values[sel], j, int(fx.num_cols), offsets)

    def to_csr(self):
        """Decode to (values float32, col_indices int64, row_splits int64)."""
        grp, rs, weights, mask = self._rec
        rec, c = np.nonzero(mask)
        rows = grp[rec] * self.GROUP + c
        cols = rs[rec]
        vals = weights[rec, c]
        order = np.lexsort((cols, rows))
        rows, cols, vals = rows[order], cols[order], vals[order]
        splits = np.zeros(self.num_rows + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows, minlength=self.num_rows), out=splits[1:])
        return vals, cols.astype(np.int64), splits


def band_from_sparse(sp, offsets: np.ndarray) -> BandOperator:
    key = ("band", tuple(int(o) for o in offsets))
    if hasattr(sp, "kept") and getattr(sp, "cols", None) is not None and np.ndim(sp.cols) == 3:
        return dev.CACHE.get(sp, key, lambda: BandOperator.from_fixed(sp, offsets))
    return dev.CACHE.get(sp, key, lambda: BandOperator.from_csr(sp.values, sp.col_indices, sp.row_splits,
                                                                int(sp.num_cols), offsets))


def band_from_dense(interp, offsets: np.ndarray) -> BandOperator:
    """Keep-all band image of a dense InterpMatrix: identical to the keep-all CSR's image."""
    def build():
        mat = np.asarray(interp.matrix)
        j, ncol = mat.shape
        rows = np.repeat(np.arange(j, dtype=np.int64), ncol)
        cols = np.tile(np.arange(ncol, dtype=np.int64), j)
        return BandOperator(rows, cols, mat.ravel(), j, ncol, offsets)
    return dev.CACHE.get(interp, ("band_dense", tuple(int(o) for o in offsets)), build)


def _band_map(op: BandOperator, samples, argmax: bool, out_map: bool):
    buf, f, batched = _lag_major(samples, op.num_cols)
    z = torch.empty((f, op.num_rows), dtype=torch.float32, device=buf.device) if out_map else None
    keys = _new_keys(f, argmax, op.num_rows)
    if op.num_rows == 0:
        return _finish(z, keys, batched, argmax)
    nat.call("srpgpu_sspi_map", dev.ptr(buf), buf.shape[1], f, op.num_cols, op.num_pairs,
             dev.ptr(op.d_tile_off), dev.ptr(op.d_blob), op.num_rows, op.max_pair_records,
             op.max_tile_records, dev.ptr(z), dev.ptr(keys), dev.stream_ptr())
    return _finish(z, keys, batched, argmax)


def _check_cols(samples, num_cols: int) -> None:
    """The reference's DimensionError check (interpolation.py:191-194) without touching data."""
    plain = isinstance(samples, (torch.Tensor, np.ndarray, list, tuple))
    vals = samples if plain else samples.values
    shape = tuple(vals.shape) if hasattr(vals, "shape") else np.shape(vals)
    if len(shape) not in (1, 2) or shape[-1] != num_cols:
        raise DimensionError(f"sample vector of shape {shape} does not match operator with "
                             f"{num_cols} columns")


# ----------------------------------------------------------------- SSPI / SI on tensor cores

ENGINES = ("auto", "tc", "tile", "tile_f16", "tile_bf16", "band")
TILE_ENGINES = {"tile": "tf32", "tile_f16": "f16", "tile_bf16": "bf16"}   # engine -> operand format
TC_MAX_COLS = 2048          # dense rows beyond this many samples: gathered windows ("tile") or band
TC_DENSITY = 12             # dense tensor cores while cols8 <= TC_DENSITY * kept entries per row
TILE_DENSITY = 4            # gathered windows while the kept entries per row are sparse


def _cols8(n: int) -> int:
    return (int(n) + 7) // 8 * 8


class DenseInterpOperator:
    """Dense bf16 hi/lo planes [2][J][cols8] of an interpolation operator (tensor-core engine).

    The sparse fit's dropped entries are zeros, so the dense product equals the sparse
    one (interpolation.py:121-126); operands are split x = bf16(x) + bf16(x - bf16(x)).
    """

    def __init__(self, mat32: np.ndarray):
        j, s = mat32.shape
        self.num_rows, self.num_cols, self.cols8 = j, s, _cols8(s)
        src = torch.from_numpy(np.ascontiguousarray(mat32, dtype=np.float32)).to(dev.device())
        self.planes = torch.empty((2, j, self.cols8), dtype=torch.bfloat16, device=src.device)
        nat.call("srpgpu_split_bf16", dev.ptr(src), s, 0, j, s, dev.ptr(self.planes), self.cols8,
                 dev.stream_ptr())


def dense_from_sparse(sp) -> DenseInterpOperator:
    def build():
        s = int(sp.num_cols)
        if np.ndim(sp.values) == 3:          # FixedNnzInterp: (P, J, k) blocks
            p_count, j, k = sp.values.shape
            keep = np.broadcast_to((np.arange(k)[None, :] < np.asarray(sp.kept)[:, None])[:, None, :],
                                   sp.values.shape)
            rows = np.broadcast_to(np.arange(j, dtype=np.int64)[None, :, None], sp.values.shape)[keep]
            cols = np.asarray(sp.cols)[keep].astype(np.int64)
            vals = np.asarray(sp.values)[keep]
        else:
            splits = np.asarray(sp.row_splits, dtype=np.int64)
            j = splits.shape[0] - 1
            rows = np.repeat(np.arange(j, dtype=np.int64), np.diff(splits))
            cols = np.asarray(sp.col_indices, dtype=np.int64)
            vals = np.asarray(sp.values)
        mat = np.zeros((j, s), dtype=np.float32)
        mat[rows, cols] = vals.astype(np.float32)
        return DenseInterpOperator(mat)
    return dev.CACHE.get(sp, "dense_bf16x2", build)


def dense_from_matrix(interp) -> DenseInterpOperator:
    return dev.CACHE.get(interp, "dense_bf16x2",
                         lambda: DenseInterpOperator(np.asarray(interp.matrix).astype(np.float32)))


# contiguous 256-candidate tiles while their MMA work stays within 3% (SRPGPU_CONTIGUOUS_SLACK overrides)
CONTIGUOUS_K_SLACK = float(os.environ.get("SRPGPU_CONTIGUOUS_SLACK", "1.03"))
CONTIGUOUS_SHORT_SLACK, CONTIGUOUS_SHORT_K = 1.6, 512.0
F16_AUTO = True             # auto: PHAT-bounded samples take the fp16x3 gathered-window engine
F16_SLAB_SCALE = 256.0      # slab weights are split as fp16(w * 256): |w| <= 1, lo stays normal down to |w| ~ 1e-3
TC_MIN_FRAMES = 0           # batches below this take the band engine (set from the cfg5 batch sweep)


def interp_engine(num_cols: int, kept_per_row: float, engine: str = "auto", frames: int | None = None,
                  pairs: bool = True, bounded: bool = False) -> str:
    """'tile' / 'tile_f16' (per-tile gathered lag windows on the tensor cores with split
    operands and fp32 chunk folds: FP32-class, the default wherever the tensor cores pay;
    'tile_f16' -- fp16 hi / lo operands, the same 22 significant bits as the 3xTF32 split at
    twice the MMA rate -- when the samples are `bounded` (PHAT: |xi| <= 2(K-1)), else 'tile'
    = 3xTF32), 'band' (tiled-band SpMM on FP32 SIMT: latency-scale sparse maps, single-pair
    operators), or the opt-in bf16x3 engines 'tc' (dense operator) and 'tile_bf16'
    (gathered windows)."""
    if engine not in ENGINES:
        raise ValueError(f"unknown engine {engine!r}")
    if engine != "auto":
        return engine
    if frames is not None and frames < TC_MIN_FRAMES:
        return "band"
    c8 = _cols8(num_cols)
    dense_ok = c8 <= TC_MAX_COLS and c8 <= TC_DENSITY * max(kept_per_row, 1.0)
    if pairs and (dense_ok or (c8 > TC_MAX_COLS and kept_per_row * TILE_DENSITY < c8)):
        return "tile_f16" if bounded and F16_AUTO else "tile"
    return "band"


class TileOperator:
    """Device image of the gathered-window operator (tiles.TileLayout) for engines "tile"
    (3xTF32: fp32 slab planes hi = tf32_rne(v), lo = tf32_rne(v - hi)), "tile_f16" (fp16 hi /
    lo planes of v * F16_SLAB_SCALE) and "tile_bf16" (bf16 hi / lo slab planes)."""

    MAX_BLOCKS = 128            # 64-lag operator blocks per tile (interp_gather_tc.cu kMaxBlocks)

    def __init__(self, sp, offsets, num_rows: int, tf32: bool = True, fmt: str | None = None):
        fmt = fmt or ("tf32" if tf32 else "bf16")
        tf32 = fmt == "tf32"
        self.fmt = fmt
        # J % 8 == 0 (cfg3 / cfg5): tiles of aligned 8-candidate runs, so the pair kernel
        # stores the map straight into grid order in whole 32-byte sectors (no tile-order
        # scratch, no gather pass; cfg3 K is even 4% smaller than with compact tiles)
        self.grid_order = fmt in ("tf32", "f16") and num_rows % 8 == 0
        lay = tiles.TileLayout(sp, offsets, num_rows, group=4 if tf32 else 8, runs=self.grid_order)
        # tiles of 256 consecutive candidates where they cost no more K (short windows: any tiling
        # pays about one lag group per pair -- cfg3 / cfg5): the pair kernel then stores the map
        # into grid order with 2D TMA boxes (whole 128-byte lines, asynchronous) instead of
        # per-thread 32-byte runs
        self.contiguous = False
        if fmt in ("tf32", "f16") and num_rows % 4 == 0 and lay.num_tiles:
            flat = tiles.TileLayout(sp, offsets, num_rows, group=4 if tf32 else 8, contiguous=True)
            k_of = (lambda l: l.mean_k_stages) if tf32 else (lambda l: l.mean_k_stages32)
            work, base = k_of(flat) * flat.num_tiles, k_of(lay) * lay.num_tiles
            # ... or up to 1.6x the K while the tiles are short (K <= 512: there the per-run stores of
            # the other layout, not the MMAs, set the pace -- cfg3: K 224 -> 310, map 0.81 -> 0.54 ms)
            cheap = work <= CONTIGUOUS_K_SLACK * base or (work <= CONTIGUOUS_SHORT_SLACK * base
                                                         and k_of(flat) <= CONTIGUOUS_SHORT_K)
            if cheap and int(flat.tile_nkb.max()) <= self.MAX_BLOCKS:
                lay, self.contiguous, self.grid_order = flat, True, True
        if lay.num_tiles and int(lay.tile_nkb.max()) > self.MAX_BLOCKS:
            raise ValueError(f"a candidate tile needs {int(lay.tile_nkb.max())} lag blocks "
                             f"(> {self.MAX_BLOCKS}): use engine 'band'")
        d = dev.device()
        self.tf32 = bool(tf32)
        self.num_rows, self.num_cols, self.cols8 = int(num_rows), int(lay.num_cols), _cols8(lay.num_cols)
        self.num_tiles, self.num_slabs = lay.num_tiles, lay.num_slabs
        # the K the kernel iterates: 16-lag stages (3xTF32), 32-lag stages (fp16x3) or 64-lag blocks (bf16)
        self.mean_k = {"tf32": lay.mean_k_stages, "f16": lay.mean_k_stages32, "bf16": lay.mean_k}[fmt]
        rows = max(1, lay.num_slabs) * tiles.HALF
        dt = {"tf32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[fmt]
        self.planes = torch.empty((2, rows, tiles.SLAB), dtype=dt, device=d)
        if lay.num_slabs:
            src = torch.from_numpy(lay.slabs.reshape(-1, tiles.SLAB)).to(d)
            if self.tf32:
                nat.call("srpgpu_split_tf32", dev.ptr(src), tiles.SLAB, dev.ptr(self.planes), tiles.SLAB,
                         src.shape[0], tiles.SLAB, dev.stream_ptr())
            elif fmt == "f16":
                nat.call("srpgpu_split_f16_rows", dev.ptr(src), tiles.SLAB, src.shape[0], tiles.SLAB, None,
                         F16_SLAB_SCALE, dev.ptr(self.planes), tiles.SLAB, rows, dev.stream_ptr())
            else:
                nat.call("srpgpu_split_bf16", dev.ptr(src), tiles.SLAB, 0, src.shape[0], tiles.SLAB,
                         dev.ptr(self.planes), tiles.SLAB, dev.stream_ptr())
            del src
        self.group_col = dev.as_i32(lay.group_col if lay.group_col.size else np.zeros(8, np.int32))
        self.tile_slab = dev.as_i32(lay.tile_slab)
        self.tile_nkb = dev.as_i32({"tf32": lay.tile_nst, "f16": lay.tile_nst32, "bf16": lay.tile_nkb}[fmt])
        self.tile_rows = dev.as_i32(lay.tile_rows)
        self.tile_pos = dev.as_i32(lay.tile_pos)
        self._layout = lay
        lay.slabs = None                      # host copy no longer needed


def tile_from_sparse(sp, offsets: np.ndarray, tf32: bool = True, fmt: str | None = None) -> TileOperator:
    fmt = fmt or ("tf32" if tf32 else "bf16")
    num_rows = int(sp.values.shape[1]) if np.ndim(sp.values) == 3 else int(np.asarray(sp.row_splits).shape[0] - 1)
    return dev.CACHE.get(sp, (f"tile_{fmt}x3", tuple(int(o) for o in offsets)),
                         lambda: TileOperator(sp, offsets, num_rows, fmt=fmt))


# Gathered-window maps straight into grid order (no untile pass): measured 2.3x SLOWER at
# cfg4 (76 vs 33.5 ms; 166 GB of DRAM reads: the L2 read-modify-writes partial 32-byte
# sectors shared between tiles), so the tile-order store + untile gather stays the default.
TILE_GRID_ORDER = False


def _tile_map(op: TileOperator, samples, offsets, argmax: bool, out_map: bool):
    planes, f, batched = sample_planes(samples, op.num_cols, natural=offsets, fmt=op.fmt)
    z = torch.empty((f, op.num_rows), dtype=torch.float32, device=planes.device) if out_map else None
    # tile-order scratch: whole 256-frame units (the pair kernels store it unit by unit)
    zt = (torch.empty(((f + 255) // 256 * 256, op.num_tiles * tiles.TILE), dtype=torch.float32, device=planes.device)
          if out_map and not (TILE_GRID_ORDER or op.grid_order) else None)
    keys = _new_keys(f, argmax)
    head = (dev.ptr(planes), f, op.num_cols, planes.shape[2], dev.ptr(op.planes), op.num_slabs,
            dev.ptr(op.group_col), dev.ptr(op.tile_slab), dev.ptr(op.tile_nkb), dev.ptr(op.tile_rows),
            op.num_tiles, op.num_rows, dev.num_sms(), None if op.contiguous else dev.ptr(op.tile_pos))
    tail = (dev.ptr(zt), dev.ptr(z), dev.ptr(keys), dev.stream_ptr())
    if op.fmt == "f16":
        nat.call("srpgpu_interp_map_gather_f16", *head, 1.0 / F16_SLAB_SCALE, *tail)
    else:
        nat.call("srpgpu_interp_map_gather_tf32" if op.tf32 else "srpgpu_interp_map_gather_tc", *head, *tail)
    return _finish(z, keys, batched, argmax)


def tile_map_stages(sp, samples, engine: str = "tile_f16"):
    """(gather, untile) callables of the CTA-pair gathered-window map's two kernels on these
    samples -- the tile-order map + argmax keys, then the gather back to grid order -- so a
    benchmark can time each on its own (`sspi_map` runs them back to back).  untile is None
    when the engine stores straight into grid order (J % 8 == 0)."""
    offsets = _sample_offsets(samples, int(sp.num_cols))
    op = tile_from_sparse(sp, offsets, fmt=TILE_ENGINES[engine])
    if op.fmt == "bf16":
        raise ValueError("tile_map_stages: the CTA-pair engines only ('tile', 'tile_f16')")
    planes, f, _ = sample_planes(samples, op.num_cols, natural=offsets, fmt=op.fmt)
    z = torch.empty((f, op.num_rows), dtype=torch.float32, device=planes.device)
    zt = None if op.grid_order else torch.empty(((f + 255) // 256 * 256, op.num_tiles * tiles.TILE),
                                                dtype=torch.float32, device=planes.device)
    keys = _new_keys(f, True)
    head = (dev.ptr(planes), f, op.num_cols, planes.shape[2], dev.ptr(op.planes), op.num_slabs,
            dev.ptr(op.group_col), dev.ptr(op.tile_slab), dev.ptr(op.tile_nkb), dev.ptr(op.tile_rows),
            op.num_tiles, op.num_rows, dev.num_sms(), None if op.contiguous else dev.ptr(op.tile_pos))

    def gather():
        tail = (dev.ptr(zt), None if zt is not None else dev.ptr(z), dev.ptr(keys), dev.stream_ptr())
        if op.fmt == "f16":
            nat.call("srpgpu_interp_map_gather_f16", *head, 1.0 / F16_SLAB_SCALE, *tail)
        else:
            nat.call("srpgpu_interp_map_gather_tf32", *head, *tail)

    def untile():
        nat.call("srpgpu_interp_map_untile", dev.ptr(zt), op.num_tiles, dev.ptr(op.tile_pos), op.num_rows, f,
                 dev.ptr(z), 1, dev.stream_ptr())

    return gather, (untile if zt is not None else None), z, keys


def sample_planes(samples, num_cols: int, natural=None, tf32: bool = False, fmt: str | None = None):
    """(planes, frames, batched) of any samples input (bf16 hi / lo; fmt "tf32": fp32 TF32
    hi / lo, "f16": fp16 hi / lo -- both natural lag-major only; fp16 needs bounded samples).

    natural None: frame-major planes [2][F][cols8] in storage column order (dense engine);
    natural = the pair offsets: lag-major planes [2][cols8][F8] in natural lag order
    (gathered-window engine).  Kernel-produced TdGccSamples may already carry them.
    """
    fmt = fmt or ("tf32" if tf32 else "bf16")
    tf32 = fmt == "tf32"
    want_nat = natural is not None
    planes = getattr(samples, "bf16_planes", None)
    c8 = _cols8(num_cols)
    if planes is not None and bool(getattr(samples, "planes_natural", False)) == want_nat and \
            getattr(samples, "planes_fmt", "bf16") == fmt and planes.shape[1 if want_nat else 2] == c8:
        vals = samples.values
        batched = vals.dim() == 2
        return planes, (vals.shape[0] if batched else 1), batched
    src = None
    if want_nat:
        key = ("natural_src_i32", tuple(int(o) for o in natural))
        src = _NAT_SRC.get(key)
        if src is None:
            src = _NAT_SRC.setdefault(key, dev.as_i32(tiles.natural_columns(np.asarray(natural))))
        buf, f, batched = _lag_major(samples, num_cols)
        if tf32:
            f32 = (f + 31) // 32 * 32
            planes = torch.empty((2, c8, f32), dtype=torch.float32, device=buf.device)
            nat.call("srpgpu_split_tf32_rows", dev.ptr(buf), buf.shape[1], num_cols, f, dev.ptr(src),
                     dev.ptr(planes), f32, c8, dev.stream_ptr())
            return planes, f, batched
        if fmt == "f16":
            f64 = (f + 63) // 64 * 64
            planes = torch.empty((2, c8, f64), dtype=torch.float16, device=buf.device)
            nat.call("srpgpu_split_f16_rows", dev.ptr(buf), buf.shape[1], num_cols, f, dev.ptr(src), 1.0,
                     dev.ptr(planes), f64, c8, dev.stream_ptr())
            return planes, f, batched
        f8 = (f + 7) // 8 * 8
        planes = torch.empty((2, c8, f8), dtype=torch.bfloat16, device=buf.device)
        nat.call("srpgpu_split_bf16_rows", dev.ptr(buf), buf.shape[1], num_cols, f, dev.ptr(src), dev.ptr(planes),
                 f8, c8, dev.stream_ptr())
        return planes, f, batched
    buf = getattr(samples, "lag_major", None)
    if buf is not None and buf.shape[0] == num_cols:
        vals = samples.values
        batched = vals.dim() == 2
        f = vals.shape[0] if batched else 1
        planes = torch.empty((2, f, c8), dtype=torch.bfloat16, device=buf.device)
        nat.call("srpgpu_split_bf16", dev.ptr(buf), buf.shape[1], 1, f, num_cols, dev.ptr(planes), c8,
                 dev.stream_ptr())
        return planes, f, batched
    x, batched = _sample_matrix(samples, num_cols)
    f = x.shape[0]
    planes = torch.empty((2, f, c8), dtype=torch.bfloat16, device=x.device)
    nat.call("srpgpu_split_bf16", dev.ptr(x), num_cols, 0, f, num_cols, dev.ptr(planes), c8, dev.stream_ptr())
    return planes, f, batched


_NAT_SRC: dict = {}


def _tc_map(op: DenseInterpOperator, samples, argmax: bool, out_map: bool):
    planes, f, batched = sample_planes(samples, op.num_cols)
    z = torch.empty((f, op.num_rows), dtype=torch.float32, device=planes.device) if out_map else None
    keys = _new_keys(f, argmax, op.num_rows)
    if op.num_rows == 0:
        return _finish(z, keys, batched, argmax)
    nat.call("srpgpu_interp_map_tc", dev.ptr(planes), f, dev.ptr(op.planes), op.num_rows, op.cols8,
             dev.ptr(z), dev.ptr(keys), dev.stream_ptr())
    return _finish(z, keys, batched, argmax)


def map_engine(variant: str, op, engine: str = "auto", frames: int | None = None, bounded: bool = False):
    """Engine sspi_map / si_map take on this operator and batch size ("tc" | "tile" |
    "tile_f16" | "band"; None for the other variants).  bounded: the samples are PHAT-weighted
    (|xi| <= 2(K-1)), so the fp16x3 engine may take the tensor-core cases."""
    if variant == "si":
        n = int(np.asarray(op.matrix).shape[1])
        return interp_engine(n, n, engine, frames, bounded=bounded)
    if variant == "sspi":
        return interp_engine(int(op.num_cols), _kept_per_row(op), engine, frames, bounded=bounded)
    return None


def plane_args(engine: str) -> dict:
    """frames_to_samples keywords that make the frontend also write the operand planes the
    map engine reads (bf16 frame-major for "tc", natural lag-major bf16 / TF32 for the
    gathered-window engines)."""
    return {"planes": engine == "tc" or engine in TILE_ENGINES, "natural": engine in TILE_ENGINES,
            "fmt": TILE_ENGINES.get(engine, "bf16")}


def uses_tc(variant: str, op, engine: str = "auto", frames: int | None = None) -> bool:
    """Whether sspi_map / si_map on this operator (and batch size) run on the tensor cores."""
    eng = map_engine(variant, op, engine, frames)
    return eng == "tc" or eng in TILE_ENGINES


F16_MAX_HALF_LEN = 16384    # PHAT samples are bounded by 2(K-1): far inside fp16's 65504 up to here


def phat_bounded(weighting: str, half_len: int) -> bool:
    """Whether samples with this weighting and frame half-length K fit fp16 operands."""
    return weighting == "phat" and int(half_len) <= F16_MAX_HALF_LEN


def _bounded(samples) -> bool:
    """Kernel-produced PHAT samples (|xi| <= 2(K-1)): safe as fp16 hi / lo operands."""
    spec = getattr(samples, "spec", None)
    return bool(getattr(samples, "phat", False)) and int(getattr(spec, "half_len", 0) or 0) <= F16_MAX_HALF_LEN


def _num_frames(samples) -> int:
    plain = isinstance(samples, (torch.Tensor, np.ndarray, list, tuple))
    vals = samples if plain else samples.values
    shape = tuple(vals.shape) if hasattr(vals, "shape") else np.shape(vals)
    return int(shape[0]) if len(shape) == 2 else 1


def _kept_per_row(sp) -> float:
    if hasattr(sp, "row_splits"):
        j = max(1, np.asarray(sp.row_splits).shape[0] - 1)
        return float(np.asarray(sp.values).shape[0]) / j
    return float(np.sum(np.asarray(sp.kept)))            # fixed-nnz: k per (row, pair)


def sspi_map(sp, samples, *, argmax: bool = False, out_map: bool = True, engine: str = "auto"):
    """Sparse interpolation map z_i = sum_{e in row i} v_e xi[c_e] (interpolation.py:188-195).

    engine "tc": the operator densified into bf16 hi/lo planes on the tensor cores
    (3 MMA passes, ~1e-6 normalized error); "tile": the same arithmetic over per-tile
    gathered lag windows (long sample vectors, BASELINE cfg4); "band": the tiled-band
    FP32 SpMM; "auto" picks by sample-vector length and sparsity.
    """
    num_cols = int(sp.num_cols)
    _check_cols(samples, num_cols)                 # reference DimensionError check first
    offsets = _sample_offsets(samples, num_cols)
    eng = interp_engine(num_cols, _kept_per_row(sp), engine, _num_frames(samples), offsets.shape[0] > 2,
                        bounded=_bounded(samples))
    if eng == "tc":
        return _tc_map(dense_from_sparse(sp), samples, argmax, out_map)
    if eng in TILE_ENGINES:
        op = tile_from_sparse(sp, offsets, fmt=TILE_ENGINES[eng])
        return _tile_map(op, samples, offsets, argmax, out_map)
    op = band_from_sparse(sp, offsets)
    return _band_map(op, samples, argmax, out_map)


def si_map(interp, samples, *, argmax: bool = False, out_map: bool = True, engine: str = "auto"):
    """Dense sampling+interpolation map z = Lambda xi (interpolation.py:129-136).

    Runs the same engine and operator image as sspi_map on the keep-all fit, so
    sspi_map(keep=all) == si_map bit for bit, as in the reference (interpolation.py:112-126).
    """
    num_cols = int(np.asarray(interp.matrix).shape[1])
    _check_cols(samples, num_cols)
    offsets = spec_offsets(interp.spec)
    if int(offsets[-1]) != num_cols:
        offsets = np.array([0, num_cols], dtype=np.int64)
    eng = interp_engine(num_cols, num_cols, engine, _num_frames(samples), offsets.shape[0] > 2,
                        bounded=_bounded(samples))
    if eng == "tc":
        return _tc_map(dense_from_matrix(interp), samples, argmax, out_map)
    if eng in TILE_ENGINES:
        sp = dev.CACHE.get(interp, "keep_all_csr", lambda: _keep_all_csr(interp))
        return _tile_map(tile_from_sparse(sp, offsets, fmt=TILE_ENGINES[eng]), samples, offsets, argmax, out_map)
    return _band_map(band_from_dense(interp, offsets), samples, argmax, out_map)


def _keep_all_csr(interp):
    """The keep-all sparse fit of a dense operator (truncate_sparse(interp, J * S): every
    entry, row-major) -- the operator si_map shares with sspi_map(keep=all)."""
    from .operators import SparseInterp
    mat = np.asarray(interp.matrix)
    j, n = mat.shape
    return SparseInterp(mat.ravel().copy(), np.tile(np.arange(n, dtype=np.int64), j),
                        np.arange(0, j * n + 1, n, dtype=np.int64), n)


# ----------------------------------------------------------------- low rank

def _slri_device(lr):
    def build():
        return (dev.as_f32(np.asarray(lr.fat, dtype=np.float64)),
                dev.as_f32(np.asarray(lr.tall, dtype=np.float64)))
    return dev.CACHE.get(lr, "slri_f32", build)


def _planes_of(mat32: np.ndarray) -> DenseInterpOperator:
    return DenseInterpOperator(mat32)


LOWRANK_TC_MIN_OUTPUTS = 1 << 24   # frames x candidates from which the tensor-core product wins


def _lowrank_engine(engine: str, outputs: int) -> str:
    """'simt': the rank-R candidate product in fp32 SIMT (the default: FP32 end to end);
    'tc': on the tensor cores with bf16 hi / lo operands (opt-in speed mode, z-write bound:
    cfg3 SLRI chain 0.88 -> 0.65 ms, normalized error up to ~2.6e-5 at low ranks)."""
    if engine not in ("auto", "tc", "simt"):
        raise ValueError(f"unknown engine {engine!r}")
    return "simt" if engine == "auto" else engine


def slri_map(lr, samples, *, argmax: bool = False, out_map: bool = True, engine: str = "auto"):
    """Low-rank interpolation map z = tall (fat xi) (interpolation.py:178-185).

    The factor product fat.xi runs in fp32; the candidate product tall.(fat xi) runs in
    fp32 SIMT ("simt", the default) or, opt-in, on the tensor cores with bf16 hi/lo
    operands ("tc", ~1e-6 - 2.6e-5 normalized error).
    """
    fat = np.asarray(lr.fat)
    buf, f, batched = _lag_major(samples, fat.shape[1])
    d_fat, d_tall = _slri_device(lr)
    r, j = fat.shape[0], d_tall.shape[0]
    work = torch.empty((17, f, r), dtype=torch.float32, device=buf.device)   # + split-K partials
    z = torch.empty((f, j), dtype=torch.float32, device=buf.device) if out_map else None
    keys = _new_keys(f, argmax)
    if _lowrank_engine(engine, f * j) == "tc":
        tp = dev.CACHE.get(lr, "slri_tall_bf16x2",
                           lambda: _planes_of(np.asarray(lr.tall, dtype=np.float64).astype(np.float32)))
        wp = torch.empty((2, f, tp.cols8), dtype=torch.bfloat16, device=buf.device)
        nat.call("srpgpu_slri_map_tc", dev.ptr(buf), buf.shape[1], f, fat.shape[1], dev.ptr(d_fat),
                 dev.ptr(tp.planes), r, tp.cols8, j, dev.ptr(work), dev.ptr(wp), dev.ptr(z), dev.ptr(keys),
                 dev.stream_ptr())
        return _finish(z, keys, batched, argmax)
    nat.call("srpgpu_slri_map", dev.ptr(buf), buf.shape[1], f, fat.shape[1], dev.ptr(d_fat),
             dev.ptr(d_tall), r, j, dev.ptr(work), dev.ptr(z), dev.ptr(keys), dev.stream_ptr())
    return _finish(z, keys, batched, argmax)


def _lr_device(lr):
    def build():
        fat = np.asarray(lr.fat, dtype=np.complex128)
        tall = np.asarray(lr.tall, dtype=np.complex128)
        r, n = fat.shape
        fat2 = np.empty((2 * r, 2 * n))
        fat2[:r, 0::2], fat2[:r, 1::2] = fat.real, -fat.imag      # Re(fat psi)
        fat2[r:, 0::2], fat2[r:, 1::2] = fat.imag, fat.real       # Im(fat psi)
        tall2 = np.concatenate([2.0 * tall.real, -2.0 * tall.imag], axis=1)
        return dev.as_f32(fat2), dev.as_f32(tall2)
    return dev.CACHE.get(lr, "lr_f32", build)


def lr_map(lr, gcc, *, argmax: bool = False, out_map: bool = True, engine: str = "auto"):
    """Low-rank SRP map z = 2 Re(tall (fat psi)) (lowrank.py:51-57).

    engine as for slri_map: "simt" (default) fp32; "tc" runs the candidate product on the tensor
    cores, "simt" in fp32.
    """
    fat = np.asarray(lr.fat)
    vals = gcc if isinstance(gcc, (torch.Tensor, np.ndarray)) else gcc.values
    v = dev.as_c64(vals)
    if v.shape[-1] != fat.shape[1] or v.dim() > 2:
        raise DimensionError(f"cross-spectrum of shape {tuple(v.shape)} does not match factor "
                             f"with {fat.shape[1]} columns")
    batched = v.dim() == 2
    v = v.reshape(-1, fat.shape[1])
    d_fat2, d_tall2 = _lr_device(lr)
    r, j, f = fat.shape[0], d_tall2.shape[0], v.shape[0]
    work = torch.empty((17, f, 2 * r), dtype=torch.float32, device=v.device)  # + split-K partials
    z = torch.empty((f, j), dtype=torch.float32, device=v.device) if out_map else None
    keys = _new_keys(f, argmax)
    if _lowrank_engine(engine, f * j) == "tc":
        tp = dev.CACHE.get(lr, "lr_tall2_bf16x2", lambda: _planes_of(d_tall2.cpu().numpy()))
        wp = torch.empty((2, f, tp.cols8), dtype=torch.bfloat16, device=v.device)
        nat.call("srpgpu_lr_map_tc", dev.ptr(v), f, fat.shape[1], dev.ptr(d_fat2), dev.ptr(tp.planes), r,
                 tp.cols8, j, dev.ptr(work), dev.ptr(wp), dev.ptr(z), dev.ptr(keys), dev.stream_ptr())
        return _finish(z, keys, batched, argmax)
    nat.call("srpgpu_lr_map", dev.ptr(v), f, fat.shape[1], dev.ptr(d_fat2), dev.ptr(d_tall2), r, j,
             dev.ptr(work), dev.ptr(z), dev.ptr(keys), dev.stream_ptr())
    return _finish(z, keys, batched, argmax)


# ----------------------------------------------------------------- conventional

def _pad4(n: int) -> int:
    return (n + 3) // 4 * 4


def _tf32_rne_host(a: np.ndarray) -> np.ndarray:
    """Round float32 values to TF32 (round-to-nearest-even), as tf32_rne in common.cuh."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).copy()
    finite = (u & 0x7F800000) != 0x7F800000
    u[finite] += np.uint32(0xFFF) + ((u[finite] >> 13) & 1)
    u &= np.uint32(0xFFFFE000)
    return u.view(np.float32)


def steering_device(srp, tf32: bool = True) -> torch.Tensor:
    """(J, ld) float32: interleaved (Re H, -Im H) per bin, row pitch padded to 16 B.

    tf32=True stores the TF32-rounded (RNE) operand of the tensor-core map.  The
    complex128 matrix (in memory, or memory-mapped from an SRPM cache) is shipped in
    row blocks as float64 and converted on the GPU (srpgpu_c128_to_steering), which
    is bit-identical to conj -> complex64 -> tf32_rne on the host.
    """
    def build():
        h = np.asarray(srp.matrix)
        j, n = h.shape
        ld = _pad4(2 * n)
        out = torch.zeros((j, ld), dtype=torch.float32, device=dev.device())
        step = max(1, (256 << 20) // max(1, 16 * n))      # 256 MB host blocks
        for r0 in range(0, j, step):
            blk = np.array(h[r0:r0 + step], dtype=np.complex128, order="C", copy=True)  # memmap -> RAM block
            src = torch.from_numpy(blk.view(np.float64)).to(out.device)
            nat.call("srpgpu_c128_to_steering", dev.ptr(src), n, blk.shape[0], n, dev.ptr(out[r0]), ld,
                     1 if tf32 else 0, dev.stream_ptr())
        return out
    return dev.CACHE.get(srp, "h2_tf32" if tf32 else "h2_f32", build)


def conv_precision(srp, precision: str = "auto", gcc=None) -> str:
    """Resolve the conventional map's arithmetic: "auto" is the parity-safe FP32-class
    mode of the operator -- 3xTF32 on the tensor cores for on-chip steering
    (steering_operator), fp32 SIMT for a stored SrpMatrix -- unless the cross-spectra
    were already rounded to TF32 by their producer (gcc_frames(tf32=True), an explicit
    upstream choice of the TF32 path).  "tf32" (one TF32 pass, ~1.5e-5 normalized error
    on maps with a source, up to ~2e-4 on peakless maps) is the opt-in speed mode; its
    error is reported next to its numbers."""
    if precision not in ("auto", "tf32", "fp32", "tf32x3"):
        raise ValueError(f"unknown precision {precision!r}")
    if precision == "auto":
        if gcc is not None and getattr(gcc, "tf32_rounded", False):
            return "tf32"
        return "fp32" if hasattr(srp, "matrix") else "tf32x3"
    return precision


def srp_map_exact(srp, gcc, *, precision: str = "auto", argmax: bool = False, out_map: bool = True):
    """Conventional SRP map z = 2 Re(H psi) (srp.py:65-71).

    precision "auto" (default): "tf32x3" for on-chip steering, "fp32" for a stored
    SrpMatrix (conv_precision); "tf32x3": tcgen05 GEMM on hi / lo TF32 operands (3 MMA
    passes, fp32 folds of the TMEM chunks), <= 5e-6 normalized error; "tf32": one
    kind::tf32 pass (opt-in speed mode, ~1.5e-5); "fp32": SIMT fp32 GEMM.
    """
    if (gcc.num_pairs, gcc.num_bins) != (srp.num_pairs, srp.num_bins):
        raise DimensionError(f"cross-spectra for {gcc.num_pairs} pairs x {gcc.num_bins} bins do not "
                             f"match a {srp.num_pairs} x {srp.num_bins} transform")
    precision = conv_precision(srp, precision, gcc)
    if precision == "tf32x3" and hasattr(srp, "matrix"):
        raise ValueError("3xTF32 is provided by the on-chip steering operator (steering_operator)")
    if not hasattr(srp, "matrix"):           # implicit operator: steering generated on chip
        if precision == "fp32":
            raise ValueError("the on-chip steering path is TF32 / 3xTF32; materialize() it for fp32")
        return _srp_map_tdoa(srp, gcc, argmax, out_map, split=(precision == "tf32x3"))
    n = srp.num_pairs * srp.num_bins
    h2 = steering_device(srp, tf32=(precision == "tf32"))
    j, ld = h2.shape
    padded = getattr(gcc, "padded", None)
    if precision == "tf32" and getattr(gcc, "tf32_rounded", False) and padded is not None \
            and padded.shape[1] == ld:
        vp, batched = padded, gcc.values.dim() == 2
        f = vp.shape[0]
    else:
        v, batched = _gcc_matrix(gcc, srp.num_pairs, srp.num_bins)
        f = v.shape[0]
        vp = None
    z = torch.empty((f, j), dtype=torch.float32, device=h2.device) if out_map else None
    keys = _new_keys(f, argmax)
    if precision == "fp32":
        if ld != 2 * n:
            h2 = h2[:, :2 * n].contiguous()
        nat.call("srpgpu_srp_map_simt", dev.ptr(v), f, n, dev.ptr(h2), j, dev.ptr(z), dev.ptr(keys),
                 dev.stream_ptr())
    else:
        if vp is None:   # round psi to TF32 and re-pitch to the operand row layout
            vp = torch.empty((f, ld), dtype=torch.float32, device=h2.device)
            nat.call("srpgpu_round_tf32", dev.ptr(v), 2 * n, dev.ptr(vp), ld, f, 2 * n,
                     dev.stream_ptr())
        ks, work = _conv_split(f, j, n)
        nat.call("srpgpu_srp_map_tc", dev.ptr(vp), ld, f, n, dev.ptr(h2), ld, j, ks, dev.ptr(work), dev.ptr(z),
                 dev.ptr(keys), dev.stream_ptr())
    return _finish(z, keys, batched, argmax)


CONV_CHUNK_FLOATS = 16 * 32      # one TMEM accumulation chunk of the tcgen05 map (16 k-blocks of 32)
CONV_SPLIT_MAX = 16


def _conv_split(frames: int, num_candidates: int, num_cols: int):
    """Split-K factor of the tensor-core conventional map: grids with fewer output tiles
    (128 candidates x 256 frames) than SMs split K into whole chunks so every SM works
    (cfg2: 56 tiles -> 2 slices; cfg1: 14 tiles -> 10); (ksplit, work buffer or None)."""
    tiles = -(-num_candidates // 128) * -(-frames // 256)
    chunks = -(-2 * num_cols // CONV_CHUNK_FLOATS)
    ks = max(1, min(dev.num_sms() // max(tiles, 1), chunks, CONV_SPLIT_MAX))
    ks = -(-chunks // -(-chunks // ks))          # slices of whole chunks, none left empty (the kernel's rule)
    if ks < 2 or frames > 65535:
        return 1, None
    return ks, torch.empty((ks, frames, num_candidates), dtype=torch.float32, device=dev.device())


def _xtab_device(op) -> torch.Tensor:
    """x[i][p] = dt_p(i) * fs as float32 (the on-chip steering generator's input)."""
    return dev.CACHE.get(op, "xtab_f32", lambda: dev.as_f32(
        np.asarray(op.tdoa.delta_t, dtype=np.float64) * float(op.frame.sample_rate)))


def _srp_map_tdoa(op, gcc, argmax: bool, out_map: bool, split: bool = False):
    n = op.num_pairs * op.num_bins
    ld = _pad4(2 * n)
    padded = getattr(gcc, "padded", None)
    if split:                              # hi / lo TF32 planes of psi
        if getattr(gcc, "tf32_rounded", False):
            raise ValueError("tf32x3 needs unrounded cross-spectra (gcc_frames(..., tf32=False))")
        if getattr(gcc, "split_planes", None) is not None:
            vp, batched = gcc.split_planes, gcc.values.dim() == 2
            f = vp.shape[0] // 2
        else:
            v, batched = _gcc_matrix(gcc, op.num_pairs, op.num_bins)
            f = v.shape[0]
            vp = torch.empty((2 * f, ld), dtype=torch.float32, device=v.device)
            nat.call("srpgpu_split_tf32", dev.ptr(v), 2 * n, dev.ptr(vp), ld, f, 2 * n, dev.stream_ptr())
    elif getattr(gcc, "tf32_rounded", False) and padded is not None and padded.shape[1] == ld:
        vp, batched = padded, gcc.values.dim() == 2
        f = vp.shape[0]
    else:
        v, batched = _gcc_matrix(gcc, op.num_pairs, op.num_bins)
        f = v.shape[0]
        vp = torch.empty((f, ld), dtype=torch.float32, device=v.device)
        nat.call("srpgpu_round_tf32", dev.ptr(v), 2 * n, dev.ptr(vp), ld, f, 2 * n, dev.stream_ptr())
    j = op.num_candidates
    xt = _xtab_device(op)
    z = torch.empty((f, j), dtype=torch.float32, device=vp.device) if out_map else None
    keys = _new_keys(f, argmax)
    ks, work = _conv_split(f, j, n)
    nat.call("srpgpu_srp_map_tdoa", dev.ptr(vp), ld, f, op.num_pairs, op.num_bins + 1, dev.ptr(xt), j,
             1 if split else 0, ks, dev.ptr(work), dev.ptr(z), dev.ptr(keys), dev.stream_ptr())
    return _finish(z, keys, batched, argmax)


# ----------------------------------------------------------------- argmax

def map_argmax(z) -> torch.Tensor:
    """Per-frame argmax of z (J,) or (F, J) on the device (first index of the max)."""
    zz = dev.as_f32(z)
    batched = zz.dim() == 2
    zz = zz.reshape(-1, zz.shape[-1])
    idx = []
    for f0 in range(0, zz.shape[0], 65535):
        part = zz[f0:f0 + 65535]
        keys = torch.empty(part.shape[0], dtype=torch.int64, device=zz.device)
        nat.call("srpgpu_argmax", dev.ptr(part), part.shape[0], part.shape[1], part.shape[1],
                 dev.ptr(keys), dev.stream_ptr())
        idx.append(decode_keys(keys)[0])
    out = torch.cat(idx)
    return out if batched else out[0]


def locate(z, grid):
    """Index and coordinates of the map maximum; ties go to the lowest index (srp.py:74-80).

    z (J,) -> (int, (3,) array); z (F, J) -> ((F,) int64 array, (F, 3) array).
    """
    shape = tuple(z.shape) if hasattr(z, "shape") else np.shape(z)
    if shape[-1:] != (grid.num_points,) or len(shape) > 2:
        raise DimensionError(f"map of length {shape} does not match grid with "
                             f"{grid.num_points} points")
    idx = map_argmax(z).cpu().numpy()
    if idx.ndim == 0:
        i = int(idx)
        return i, np.asarray(grid.points)[i].copy()
    return idx, np.asarray(grid.points)[idx].copy()


def evaluate_map(kind, op, spec, frame, gcc, path="ifft", **kw):
    """Backend dispatch of the reference (cli.py:170-180); the GPU always samples by iFFT."""
    from .sampling import td_gcc_samples
    if kind == "conv":
        return srp_map_exact(op, gcc, **kw)
    if kind == "lr":
        return lr_map(op, gcc, **kw)
    if path not in ("auto", "ifft", "matrix"):
        raise ValueError(f"unknown sampling path {path!r}")
    xi = td_gcc_samples(gcc, spec, "ifft")
    if kind == "si":
        return si_map(op, xi, **kw)
    if kind == "slri":
        return slri_map(op, xi, **kw)
    if kind == "sspi":
        return sspi_map(op, xi, **kw)
    raise ValueError(f"unknown map kind {kind!r}")


# ----------------------------------------------------------------- fused chain (SSPI)

FUSED_MAX_NNZ = 32            # widest sparse row the fused chain takes (its cost grows with nnz)
FUSED_PAD = 16                # sliced-ELL chunk width of the kernel's unrolled path (kMapW)
FUSED_MAX_FRAMES_PER_SM = 8   # latency-scale batches only (a warp per frame, one wave)
FUSED_FRAME_LENS = (256, 512, 1024)


def sell_layout(sp):
    """Host image of the sliced-ELL operator: (cols [rows][32] uint16 sample index, vals
    [rows][32] float32 weight, chunk_off [ceil(J/32) + 1] int64).  Candidates come in chunks
    of 32; chunk c has width W_c = its longest row (padded to FUSED_PAD / 2 FUSED_PAD for the
    kernel's unrolled path), entries stored [row][lane]; candidate i's k-th CSR entry is row
    chunk_off[i // 32] + k, lane i % 32; padding entries have weight 0 and sample index 0."""
    splits = np.asarray(sp.row_splits, dtype=np.int64)
    cols = np.asarray(sp.col_indices, dtype=np.int64)
    vals = np.asarray(sp.values, dtype=np.float64)
    j = splits.shape[0] - 1
    nnz = np.diff(splits)
    nch = (j + 31) // 32
    width = np.zeros(nch * 32, dtype=np.int64)
    width[:j] = nnz
    width = width.reshape(nch, 32).max(axis=1)
    # chunks up to FUSED_PAD (2 FUSED_PAD) entries wide are padded to exactly FUSED_PAD
    # (2 FUSED_PAD): the kernel then loads them unconditionally at fixed offsets
    # (frontend_warp.cu kMapW)
    width = np.where(width <= FUSED_PAD, FUSED_PAD, np.where(width <= 2 * FUSED_PAD, 2 * FUSED_PAD, width))
    off = np.zeros(nch + 1, dtype=np.int64)
    np.cumsum(width, out=off[1:])
    rows = int(off[-1])
    c = np.zeros((max(rows, 1), 32), dtype=np.uint16)
    v = np.zeros((max(rows, 1), 32), dtype=np.float32)
    cand = np.repeat(np.arange(j, dtype=np.int64), nnz)
    slot = np.arange(cols.shape[0], dtype=np.int64) - np.repeat(splits[:-1], nnz)
    c[off[cand // 32] + slot, cand % 32] = cols
    v[off[cand // 32] + slot, cand % 32] = vals.astype(np.float32)
    return c, v, off


class SellOperator:
    """Device image of sell_layout for the fused frames -> SSPI map chain."""

    def __init__(self, sp):
        c, v, off = sell_layout(sp)
        nnz = np.diff(np.asarray(sp.row_splits, dtype=np.int64))
        d = dev.device()
        self.num_rows, self.num_cols = nnz.shape[0], int(sp.num_cols)
        self.max_row_nnz = int(nnz.max()) if nnz.size else 0
        self.padding = int(off[-1]) * 32 / max(1, int(nnz.sum()))
        self.cols = torch.from_numpy(c.view(np.int16)).to(d)
        self.vals = torch.from_numpy(v).to(d)
        self.chunk_off = torch.from_numpy(off.astype(np.int32)).to(d)


def sell_from_sparse(sp) -> SellOperator:
    return dev.CACHE.get(sp, "sell", lambda: SellOperator(sp))


def fused_eligible(sp, frame, spec, frames: int, num_channels: int) -> bool:
    """Whether frames_to_sspi_map takes this operator / frame shape / batch (the pipeline's
    choice for latency-scale batches: cfg1 / cfg2)."""
    if not hasattr(sp, "row_splits") or int(sp.num_cols) != int(spec_offsets(spec)[-1]):
        return False
    nnz = np.diff(np.asarray(sp.row_splits))
    if nnz.size == 0 or int(nnz.max()) > FUSED_MAX_NNZ:
        return False
    return _fused_shape_ok(frame, spec, frames, num_channels, 4 * ((nnz.size + 31) // 32 + 1))


def _fused_shape_ok(frame, spec, frames: int, num_channels: int, extra_smem: int) -> bool:
    if frame.frame_len not in FUSED_FRAME_LENS or frames > FUSED_MAX_FRAMES_PER_SM * dev.num_sms():
        return False
    s_tot = int(spec_offsets(spec)[-1])
    if s_tot > 4096:
        return False
    k = frame.frame_len // 2
    lp = frame.frame_len // 32
    smem = 4 * ((num_channels * (k + 1) + (32 // lp) * 32 * (lp + 1)) * 8) + 16 * s_tot + 8 * 1024 + extra_smem
    return smem <= 220 * 1024


def fused_slri_eligible(lr, frame, spec, frames: int, num_channels: int) -> bool:
    """Whether frames_to_slri_map takes this factorization / frame shape / batch."""
    fat = np.asarray(lr.fat)
    if fat.ndim != 2 or fat.shape[1] != int(spec_offsets(spec)[-1]):
        return False
    return _fused_shape_ok(frame, spec, frames, num_channels, 16 * fat.shape[0])


def _fused_call(name, samples, frame, pairs, spec, frames, weighting, floor, num_cols, num_rows, op_args,
                argmax, out_map):
    from . import frontend as fe
    from .sampling import _spec_device
    x = fe._signal(samples)
    if x.shape[0] != pairs.num_mics:
        raise DimensionError(f"expected {pairs.num_mics} channels, got {x.shape[0]}")
    if spec.num_pairs != pairs.num_pairs or spec.half_len != frame.half_len:
        raise DimensionError("sample spec does not match the pairs / frame")
    s_tot = int(spec_offsets(spec)[-1])
    if num_cols != s_tot:
        raise DimensionError(f"operator with {num_cols} columns does not match {s_tot} samples")
    first, count, batched = fe._frame_range(frames, fe.num_frames(frame, x.shape[1]))
    fe._check_range(frame, first, count, x.shape[1])
    w, mode, fval = fe._floor_args(weighting, floor)
    counts, offsets = _spec_device(spec)
    z = torch.empty((count, num_rows), dtype=torch.float32, device=x.device) if out_map else None
    idx = torch.empty(count, dtype=torch.int64, device=x.device) if argmax else None
    nat.call(name, dev.ptr(x), x.shape[0], x.shape[1], x.shape[1], dev.ptr(fe._window_device(frame)),
             frame.frame_len, frame.hop, first, count, dev.ptr(fe._pairs_device(pairs)), pairs.num_pairs, w, mode,
             fval, dev.ptr(counts), dev.ptr(offsets), s_tot, *op_args, num_rows, dev.ptr(z), dev.ptr(idx), None,
             dev.stream_ptr())
    zz = None if z is None else (z if batched else z[0])
    if not argmax:
        return zz
    return zz, (idx if batched else idx[0])


def frames_to_slri_map(lr, samples, frame, pairs, spec, frames=None, weighting: str = "phat", floor=None,
                       *, argmax: bool = True, out_map: bool = True):
    """The SLRI chain in one kernel: stft_frame -> fd_gcc -> td_gcc_samples -> slri_map ->
    locate (interpolation.py:178-185 for the map): y = fat . xi per frame in shared
    memory, z = tall . y, fp32.  Returns z (F, J) (None without out_map) and the argmax."""
    d_fat, d_tall = _slri_device(lr)
    def build_t():
        r16 = (d_tall.shape[1] + 15) // 16 * 16
        t = torch.zeros((r16, d_tall.shape[0]), dtype=torch.float32, device=d_tall.device)
        t[:d_tall.shape[1]] = d_tall.t()
        return t
    tall_t = dev.CACHE.get(lr, "slri_tall_t16", build_t)
    r, j = d_fat.shape[0], d_tall.shape[0]
    return _fused_call("srpgpu_frames_to_slri_map", samples, frame, pairs, spec, frames, weighting, floor,
                       int(d_fat.shape[1]), j, (dev.ptr(d_fat), dev.ptr(tall_t), r), argmax, out_map)


def frames_to_sspi_map(sp, samples, frame, pairs, spec, frames=None, weighting: str = "phat", floor=None,
                       *, argmax: bool = True, out_map: bool = True):
    """The SSPI chain in one kernel: stft_frame -> fd_gcc -> td_gcc_samples -> sspi_map ->
    locate over a range of frames (frontend.py:89-160, sampling.py:106-134,
    interpolation.py:188-195, srp.py:74-80).  The TD-GCC samples stay in shared memory.
    Returns z (F, J) (None without out_map) and, with argmax, the per-frame argmax (F,)."""
    op = sell_from_sparse(sp)
    return _fused_call("srpgpu_frames_to_sspi_map", samples, frame, pairs, spec, frames, weighting, floor,
                       op.num_cols, op.num_rows, (dev.ptr(op.cols), dev.ptr(op.vals), dev.ptr(op.chunk_off)),
                       argmax, out_map)
