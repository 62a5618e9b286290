"""Gathered-window operator layout for the tensor-core SSPI engine on long sample vectors.

When the sample vector is long (BASELINE cfg4: S = 7028 lags over 120 pairs) the dense
operator rows of `interp_tc` would cost S MACs per candidate against ~240 kept entries.
Here the candidates are cut into tiles of 256 (two MMA halves of 128 rows that share
every gathered sample tile) that are compact in TDOA space (recursive bisection along
the pair with the widest spread), and each tile only sees the union of its candidates'
kept lag windows, pair by pair, rounded up to groups of 8 consecutive lags:

    K(tile) = sum_p g * ceil(w_p / g),   w_p = width of the tile's window of pair p

with g = 8 lags for the bf16 / fp16 kernels (their MN atoms are 8 rows) and g = 4 for the 3xTF32
kernel (the tf32 MN layout has 4-row atoms): cfg4 (fixed fit) 1160 / 966 on average for
256-candidate tiles, against S = 7028.  The
tile's operator is stored dense over that K in 64-lag blocks, each block as two slabs
(`[2 * block + half][128 rows][64]`, zero where a candidate does not keep the lag), and
the kernel gathers each 8-lag group as 8 rows of the lag-major samples.
The samples live in *natural* lag order per pair (-N_p .. N_p), so a window is a
contiguous run of lag rows.

Everything here is host-side layout (the same entries as the reference's sparse
operator, interpolation.py:68-90 / 155-175, just placed differently).
"""

from __future__ import annotations

import numpy as np

TILE, HALF, GROUP, SLAB, STAGE = 256, 128, 8, 64, 16


def natural_columns(offsets: np.ndarray) -> np.ndarray:
    """perm[c_nat] = storage column: natural order -N..N per pair from 0..N, -N..-1."""
    offsets = np.asarray(offsets, dtype=np.int64)
    out = np.empty(int(offsets[-1]), dtype=np.int64)
    for p in range(offsets.shape[0] - 1):
        o, w = int(offsets[p]), int(offsets[p + 1] - offsets[p])
        n = (w - 1) // 2
        lags = np.arange(-n, n + 1)
        out[o:o + w] = o + np.where(lags >= 0, lags, w + lags)
    return out


def to_natural(cols: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    """Storage column -> natural column (same pair block)."""
    offsets = np.asarray(offsets, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    pair = np.searchsorted(offsets, cols, side="right") - 1
    base = offsets[pair]
    n = (offsets[pair + 1] - base - 1) // 2
    d = cols - base
    return base + np.where(d <= n, n + d, d - n - 1)


def _entries(sp, offsets):
    """(rows, pairs, natural cols, values f32) of every kept entry of a sparse operator."""
    if hasattr(sp, "kept") and np.ndim(getattr(sp, "cols", None)) == 3:    # FixedNnzInterp
        p_count, j, k = sp.values.shape
        keep = np.arange(k)[None, :] < np.asarray(sp.kept)[:, None]
        sel = np.broadcast_to(keep[:, None, :], sp.values.shape)
        rows = np.broadcast_to(np.arange(j, dtype=np.int64)[None, :, None], sp.values.shape)[sel]
        cols = np.asarray(sp.cols)[sel].astype(np.int64)
        vals = np.asarray(sp.values)[sel].astype(np.float32)
    else:
        splits = np.asarray(sp.row_splits, dtype=np.int64)
        rows = np.repeat(np.arange(splits.shape[0] - 1, dtype=np.int64), np.diff(splits))
        cols = np.asarray(sp.col_indices, dtype=np.int64)
        vals = np.asarray(sp.values).astype(np.float32)
    pairs = np.searchsorted(np.asarray(offsets, dtype=np.int64), cols, side="right") - 1
    return rows, pairs, to_natural(cols, offsets), vals


def bisect_tiles(feat: np.ndarray, tile: int = TILE, weight=None, lo=None, hi=None, group: int = GROUP,
                 tries: int = 1) -> list:
    """Recursive bisection of the rows of `feat` (n, D) into groups of total weight <=
    `tile` (weight: rows per item, default 1), splitting at a multiple of `tile` near the
    (weighted) median.  The split axis is the widest coordinate, or -- with the items'
    per-pair lag windows `lo` / `hi` (n, D) and tries > 1 -- the one among the `tries`
    widest whose two halves have the smallest summed window widths (rounded up to `group`
    lags, each half weighted by its share of tiles): the K the kernel iterates."""
    w = np.ones(feat.shape[0], dtype=np.int64) if weight is None else np.asarray(weight, dtype=np.int64)

    def cost(ix):
        width = hi[ix].max(axis=0) - lo[ix].min(axis=0) + 1
        return float(np.sum((width + group - 1) // group * group))

    out, stack = [], [np.arange(feat.shape[0], dtype=np.int64)]
    while stack:
        idx = stack.pop()
        total = int(w[idx].sum())
        if total <= tile or idx.shape[0] == 1:
            out.append(np.sort(idx))
            continue
        sub = feat[idx]
        spread = sub.max(axis=0) - sub.min(axis=0)
        target = tile * max(1, int(round(total / (2 * tile)))) if total > 2 * tile else total // 2
        axes = [int(np.argmax(spread))] if tries <= 1 or lo is None else list(np.argsort(-spread)[:tries])
        best = None
        for p in axes:
            order = idx[np.argsort(sub[:, p], kind="stable")]
            cum = np.cumsum(w[order])
            n1 = int(np.clip(np.searchsorted(cum, target, side="right"), 1, idx.shape[0] - 1))
            if len(axes) == 1:
                best = (0.0, order[:n1], order[n1:])
                break
            a, b = order[:n1], order[n1:]
            c = cost(a) * (w[a].sum() / tile) + cost(b) * (w[b].sum() / tile)
            if best is None or c < best[0]:
                best = (c, a, b)
        stack.append(best[2])
        stack.append(best[1])
    return out


BISECT_TRIES = 8     # split axes tried per bisection step (1: widest only; 8: -4% window K at cfg4)


class TileLayout:
    """Host image of the gathered-window operator (see the module docstring).

    slabs      (2 * num_blocks, 128, 64) float32 operator values: block b, half h -> 2b + h
    group_col  (num_blocks * 64 / group,) int32: first natural sample index (lag row) of each
               group of `group` lags
    tile_slab  (T,) int32 first 64-lag block of each tile; tile_nkb (T,) blocks per tile;
               tile_nst (T,) 16-lag stages per tile (what the 3xTF32 kernel iterates);
               tile_nst32 (T,) 32-lag stages per tile (the fp16x3 kernel)
    tile_rows  (T, 256) int32 candidate of each tile row (ascending; -1 = padding);
               rows 0-127 are half 0, 128-255 half 1
    tile_pos   (J,) int32 position t * 256 + row of each candidate (the kernel writes the map
               in this tile order, fully coalesced; a gather pass restores grid order)
    """

    def __init__(self, sp, offsets, num_rows: int, group: int = GROUP, runs: bool = False,
                 contiguous: bool = False):
        """contiguous: tile t = candidates 256 t .. 256 t + 255 (the kernel stores the map
        straight into grid order with 2D TMA boxes; worth it where the windows are so short
        that any tiling pays one lag group per pair, cfg3 / cfg5).
        runs: tiles made of aligned runs of 8 consecutive candidates (each run one 32-byte
        sector of a map row when J % 8 == 0), 8 tile rows per run in ascending order, so
        the kernel can store the map straight into grid order with whole sectors (no
        tile-order scratch, no gather pass); otherwise tiles of compact candidates."""
        if group not in (4, 8):
            raise ValueError("lag groups of 4 (tf32 kernel) or 8 (bf16 kernel)")
        self.group = int(group)
        self.contiguous = bool(contiguous)
        self.runs = bool(runs) and not self.contiguous
        GROUP = self.group
        offsets = np.asarray(offsets, dtype=np.int64)
        p_count = offsets.shape[0] - 1
        rows, pairs, ncol, vals = _entries(sp, offsets)
        self.num_rows, self.num_cols, self.num_pairs = int(num_rows), int(offsets[-1]), p_count
        # per (candidate, pair): window of kept natural columns -> bisection features
        key = rows * p_count + pairs
        lo_ip = np.full(num_rows * p_count, np.iinfo(np.int64).max)
        hi_ip = np.full(num_rows * p_count, -1)
        np.minimum.at(lo_ip, key, ncol)
        np.maximum.at(hi_ip, key, ncol)
        empty = hi_ip < 0
        feat = ((lo_ip + hi_ip) * 0.5).astype(np.float32).reshape(num_rows, p_count)
        if empty.any():
            centre = ((offsets[:-1] + offsets[1:] - 1) * 0.5).astype(np.float32)
            feat = np.where(empty.reshape(num_rows, p_count), centre[None, :], feat)
        tile_of = np.zeros(num_rows, dtype=np.int64)
        row_of = np.zeros(num_rows, dtype=np.int64)
        if self.contiguous:
            t_count = (num_rows + TILE - 1) // TILE
            tile_rows = np.full((t_count, TILE), -1, dtype=np.int32)
            cand = np.arange(num_rows)
            tile_of, row_of = cand // TILE, cand % TILE
            tile_rows[tile_of, row_of] = cand
        elif self.runs and num_rows:
            n_runs = (num_rows + 7) // 8
            imax = np.iinfo(np.int64).max
            pad = n_runs * 8 - num_rows
            f3 = np.concatenate([feat, np.repeat(feat[-1:], pad, axis=0)]).reshape(n_runs, 8, p_count)
            lo3 = np.concatenate([np.where(empty, imax, lo_ip).reshape(num_rows, p_count),
                                  np.full((pad, p_count), imax)]).reshape(n_runs, 8, p_count)
            hi3 = np.concatenate([hi_ip.reshape(num_rows, p_count),
                                  np.full((pad, p_count), -1)]).reshape(n_runs, 8, p_count)
            # a run that wraps around the grid's fastest axis holds two far-apart clusters (its
            # candidates before / after the wrap): one jump between neighbours dwarfs the others
            d = np.abs(np.diff(f3, axis=1)).max(axis=2)                              # (n_runs, 7)
            ks = d.argmax(axis=1)
            jump = d[np.arange(n_runs), ks]
            d[np.arange(n_runs), ks] = -1.0
            wraps = (jump > 4.0) & (jump > 4.0 * d.max(axis=1))
            head = np.arange(8)[None, :] < np.where(wraps, ks + 1, 8)[:, None]       # candidates before the wrap

            def part(mask):
                m3 = mask[:, :, None]
                cnt = np.maximum(1, mask.sum(axis=1))[:, None]
                rf = (np.where(m3, f3, 0.0).sum(axis=1) / cnt).astype(np.float32)
                rl = np.where(m3, lo3, imax).min(axis=1)
                rh = np.where(m3, hi3, -1).max(axis=1)
                return rf, np.where(rh < 0, 0, rl), rh

            hf, hl, hh = part(head)
            tf_, tl, th = part(~head)
            tiles = []
            plain = np.flatnonzero(~wraps)
            if plain.size:
                tiles += [plain[ix] for ix in bisect_tiles(hf[plain], TILE, weight=np.full(plain.size, 8),
                                                           lo=hl[plain], hi=hh[plain], group=GROUP,
                                                           tries=BISECT_TRIES)]
            wrapped = np.flatnonzero(wraps)
            if wrapped.size:      # bisected on both clusters' windows (2P coordinates)
                tiles += [wrapped[ix] for ix in
                          bisect_tiles(np.concatenate([hf[wrapped], tf_[wrapped]], axis=1), TILE,
                                       weight=np.full(wrapped.size, 8),
                                       lo=np.concatenate([hl[wrapped], tl[wrapped]], axis=1),
                                       hi=np.concatenate([hh[wrapped], th[wrapped]], axis=1), group=GROUP,
                                       tries=BISECT_TRIES)]
            self.num_wrapped_runs = int(wrapped.size)
            t_count = len(tiles)
            tile_rows = np.full((t_count, TILE), -1, dtype=np.int32)
            for t, rr in enumerate(tiles):
                cand = (np.sort(rr)[:, None] * 8 + np.arange(8)[None, :]).ravel()
                pos = np.arange(cand.shape[0])
                ok = cand < num_rows
                tile_rows[t, pos[ok]] = cand[ok]
                tile_of[cand[ok]] = t
                row_of[cand[ok]] = pos[ok]
        else:
            clo = np.where(empty, 0, lo_ip).reshape(num_rows, p_count)
            chi = hi_ip.reshape(num_rows, p_count)
            tiles = bisect_tiles(feat, lo=clo, hi=chi, group=GROUP, tries=BISECT_TRIES) if num_rows else []
            t_count = len(tiles)
            tile_rows = np.full((t_count, TILE), -1, dtype=np.int32)
            for t, idx in enumerate(tiles):
                tile_rows[t, :idx.shape[0]] = idx
                tile_of[idx] = t
                row_of[idx] = np.arange(idx.shape[0])
        # per (tile, pair): the kept lags of the tile's candidates, covered greedily by groups of
        # GROUP consecutive lags (each group is gathered on its own, so a tile may hold several
        # disjoint windows of a pair -- the two clusters of wrapped runs -- and skips the holes)
        big = np.int64(self.num_cols + GROUP + 1)
        tp_e = tile_of[rows] * p_count + pairs                                    # (tile, pair) of each entry
        comb = np.unique(tp_e * big + ncol)                                       # distinct (tile, pair, lag), sorted
        n_tp = t_count * p_count
        ptr = np.searchsorted(comb, np.arange(n_tp, dtype=np.int64) * big)        # first lag of each (tile, pair)
        end = np.searchsorted(comb, (np.arange(n_tp, dtype=np.int64) + 1) * big)
        g_key, g_start = [], []
        live = np.flatnonzero(ptr < end)
        while live.size:
            start = comb[ptr[live]]                                               # key * big + first uncovered lag
            g_key.append(live)
            g_start.append(start)
            ptr[live] = np.searchsorted(comb, start + GROUP)
            live = live[ptr[live] < end[live]]
        if g_key:
            g_comb = np.sort(np.concatenate(g_start))                             # groups in (tile, pair, lag) order
        else:
            g_comb = np.zeros(0, dtype=np.int64)
        g_tp = g_comb // big
        ngroups = np.bincount(g_tp, minlength=n_tp).reshape(t_count, p_count)     # (T, P)
        tile_groups = ngroups.sum(axis=1)
        tile_nkb = np.maximum(1, (tile_groups * GROUP + SLAB - 1) // SLAB)
        tile_nst = np.maximum(1, (tile_groups * GROUP + STAGE - 1) // STAGE)   # 16-lag stages (tf32 kernel)
        tile_nst32 = np.maximum(1, (tile_groups * GROUP + 2 * STAGE - 1) // (2 * STAGE))   # 32-lag stages (fp16 kernel)
        tile_slab = np.zeros(t_count, dtype=np.int64)
        if t_count:
            tile_slab[1:] = np.cumsum(tile_nkb)[:-1]
        num_blocks = int(tile_nkb.sum()) if t_count else 0
        # groups are sorted by (tile, pair, lag): group i of tile t sits at slot
        # tile_slab[t] * (SLAB // GROUP) + (i - first group of t)
        g_tile = g_tp // p_count
        tile_g0 = np.zeros(t_count + 1, dtype=np.int64)
        tile_g0[1:] = np.cumsum(tile_groups)
        g_slot = tile_slab[g_tile] * (SLAB // GROUP) + (np.arange(g_comb.shape[0]) - tile_g0[g_tile])
        group_col = np.zeros(num_blocks * (SLAB // GROUP), dtype=np.int64)
        group_col[g_slot] = g_comb % big
        # scatter the entries into the slabs
        g_e = np.searchsorted(g_comb, tp_e * big + ncol, side="right") - 1        # group of each entry
        t_e = tile_of[rows]
        kpos = (g_e - tile_g0[t_e]) * GROUP + (ncol - g_comb[g_e] % big)
        r_e = row_of[rows]
        slab = 2 * (tile_slab[t_e] + kpos // SLAB) + r_e // HALF
        self.slabs = np.zeros((2 * num_blocks, HALF, SLAB), dtype=np.float32)
        self.slabs[slab, r_e % HALF, kpos % SLAB] = vals
        self.group_col = group_col.astype(np.int32)
        self.tile_slab = tile_slab.astype(np.int32)
        self.tile_nkb = tile_nkb.astype(np.int32)
        self.tile_nst = tile_nst.astype(np.int32)
        self.tile_nst32 = tile_nst32.astype(np.int32)
        self.tile_rows = tile_rows
        self.tile_pos = (tile_of * TILE + row_of).astype(np.int32)
        self.num_tiles = t_count
        self.num_blocks = num_blocks
        self.num_slabs = 2 * num_blocks
        self.mean_k = float(tile_nkb.mean() * SLAB) if t_count else 0.0
        self.mean_k_stages = float(tile_nst.mean() * STAGE) if t_count else 0.0
        self.mean_k_stages32 = float(tile_nst32.mean() * 2 * STAGE) if t_count else 0.0

    def emulate(self, xi_nat: np.ndarray) -> np.ndarray:
        """float64 reference of the gathered product (test helper): z (F, J)."""
        f = xi_nat.shape[0]
        z = np.zeros((f, self.num_rows))
        g = self.group
        pad = np.concatenate([xi_nat, np.zeros((f, SLAB + g))], axis=1)
        per = SLAB // g
        for t in range(self.num_tiles):
            b0, nk = int(self.tile_slab[t]), int(self.tile_nkb[t])
            cols = self.group_col[b0 * per:(b0 + nk) * per][:, None] + np.arange(g)[None, :]
            x = pad[:, cols.ravel()]                                     # (F, nk*64)
            for h in range(2):
                a = self.slabs[2 * b0 + h:2 * (b0 + nk):2].transpose(1, 0, 2).reshape(HALF, nk * SLAB)
                r = self.tile_rows[t, h * HALF:(h + 1) * HALF]
                ok = r >= 0
                z[:, r[ok]] = (x @ a.astype(np.float64).T)[:, ok]
        return z
