"""Frame- and candidate-partitioned execution across GPUs (one process per GPU).

The reference evaluates frames serially (cli.py:241-258) and each frame and
each candidate row is independent (srp.py:71, interpolation.py:116-126), so the
path shards without any data-path exchange:

* frame partition (default): rank r maps a contiguous block of frames with a
  replicated operator; the only collective is an all-gather of the 8-byte
  packed argmax key per frame (NCCL over NVLink on GPUs, gloo in CPU tests).
* candidate partition (grids too large for one GPU's operator): rank r owns a
  contiguous block of candidate rows and all frames; per-frame keys are
  combined with an all-reduce MAX.  Keys are stored as int64 with the sign bit
  flipped so signed MAX gives the unsigned order (largest value, lowest index).

Maps stay on the GPU that computed them.

`candidate_block` cuts an operator to a contiguous block of candidate rows (the same
entries the reference would use for those rows: srp.py:51-62 row by row, the CSR rows of
interpolation.py:155-175) and `CandidateShard` runs one rank's block as a MapPipeline
whose per-frame (value, index) become global keys combined by `reduce_candidate_keys`.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

_SIGN = -(1 << 63)


def partition(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block (first, count) of `total` items for `rank` of `world`."""
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def keys_to_signed(keys: torch.Tensor) -> torch.Tensor:
    """Packed uint64 keys (stored in int64) -> order-preserving signed int64."""
    return keys ^ _SIGN


def signed_to_keys(vals: torch.Tensor) -> torch.Tensor:
    return vals ^ _SIGN


def offset_keys(keys: torch.Tensor, row_offset: int) -> torch.Tensor:
    """Re-base the candidate index packed in keys computed on a row block."""
    if row_offset == 0:
        return keys
    low = keys & 0xFFFFFFFF
    return (keys - low) | ((low - row_offset) & 0xFFFFFFFF)


def gather_frame_keys(local_keys: torch.Tensor, total_frames: int, group=None) -> torch.Tensor:
    """All-gather per-frame keys of a frame-partitioned run -> (total_frames,) on every rank."""
    world = dist.get_world_size(group)
    counts = [partition(total_frames, world, r)[1] for r in range(world)]
    width = max(counts) if counts else 0
    buf = torch.zeros(width, dtype=torch.int64, device=local_keys.device)
    buf[:local_keys.shape[0]] = local_keys
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    return torch.cat([o[:c] for o, c in zip(out, counts)])


def pipelined_steps(steps, n: int, total_frames: int, outs=None, group=None):
    """Run n steps of a frame-partitioned pipeline, all-gathering each step's per-frame
    result (8 bytes per frame, equal frame counts per rank) asynchronously.

    `steps[i % len(steps)]()` enqueues step i and returns its (F_local,) int64 result on
    the current stream.  Step i's all-gather overlaps step i+1; before step i the stream
    waits for gather i-2, whose output buffer (a ring of two) and input step slot
    (`len(steps) >= 2`) are then reused.  Returns the two output buffers; after the call
    the stream has waited for every gather.  Single process: no collective.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world > 1 and len(steps) < 2:
        raise ValueError("pipelined gathers need at least two step slots")
    works = []
    for i in range(n):
        if len(works) >= 2:
            works[-2].wait()
        res = steps[i % len(steps)]()
        if world > 1:
            if outs is None:
                outs = [torch.empty(total_frames, dtype=res.dtype, device=res.device) for _ in range(2)]
            works.append(dist.all_gather_into_tensor(outs[i % 2], res, group=group, async_op=True))
    for w in works:
        w.wait()
    return outs


def candidate_block(op, first: int, count: int):
    """The operator restricted to candidate rows [first, first + count).

    SteeringTdoa (on-chip conventional steering): the TDOA table's rows; SparseInterp (the
    reference CSR): its rows, column indices unchanged; FixedNnzInterp: its (P, J, k) rows.
    Values are the very entries of the full operator, so a block map equals the full map's
    columns bit for bit on the row-local engines.
    """
    import numpy as np
    from .operators import FixedNnzInterp, SparseInterp, SteeringTdoa
    from .scene import TdoaTable
    if isinstance(op, SteeringTdoa):
        t = op.tdoa
        return SteeringTdoa(tdoa=TdoaTable(np.ascontiguousarray(t.delta_t[first:first + count]), t.limits),
                            frame=op.frame)
    if isinstance(op, SparseInterp):
        splits = np.asarray(op.row_splits, dtype=np.int64)
        a, b = int(splits[first]), int(splits[first + count])
        return SparseInterp(np.asarray(op.values)[a:b], np.asarray(op.col_indices)[a:b],
                            splits[first:first + count + 1] - a, int(op.num_cols))
    if isinstance(op, FixedNnzInterp):
        return FixedNnzInterp(values=np.ascontiguousarray(op.values[:, first:first + count]),
                              cols=np.ascontiguousarray(op.cols[:, first:first + count]), kept=op.kept,
                              num_cols=op.num_cols)
    raise TypeError(f"no candidate partition for {type(op).__name__}")


def block_keys(z: torch.Tensor, index: torch.Tensor, row_offset: int) -> torch.Tensor:
    """Global packed keys of a block map: the kernel's per-frame argmax (first maximum of
    the block) and its value, re-based to the block's first global candidate."""
    f = index.shape[0]
    vals = z.reshape(f, -1).gather(1, index.reshape(f, 1)).reshape(f)
    return encode_host_keys(vals, index + row_offset)


class CandidateShard:
    """One rank of a candidate-partitioned map: a contiguous block of candidate rows for
    every frame of the batch (MapPipeline on `candidate_block`), whose per-frame keys are
    all-reduced (MAX) into the global first maximum (srp.py:74-80) every step."""

    def __init__(self, variant, op, frame, pairs, spec, frames: int, rank: int, world: int, **kw):
        from .pipeline import MapPipeline
        j = op.num_candidates if hasattr(op, "num_candidates") else (
            op.values.shape[1] if getattr(op, "values", None) is not None and op.values.ndim == 3
            else int(len(op.row_splits) - 1))
        self.first, self.count = partition(j, world, rank)
        self.block = candidate_block(op, self.first, self.count)
        self.pipe = MapPipeline(variant, self.block, frame, pairs, spec, frames=frames, **kw)
        self.input = self.pipe.input

    def step(self, group=None) -> torch.Tensor:
        """Replay the block's chain; -> global packed keys (frames,) on every rank."""
        z, idx = self.pipe.replay()
        keys = block_keys(z, idx, self.first)
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            keys = reduce_candidate_keys(keys, group)
        return keys


def reduce_candidate_keys(local_keys: torch.Tensor, group=None) -> torch.Tensor:
    """All-reduce MAX of per-frame keys of a candidate-partitioned run."""
    vals = keys_to_signed(local_keys.clone())
    dist.all_reduce(vals, op=dist.ReduceOp.MAX, group=group)
    return signed_to_keys(vals)


def decode_host_keys(keys: torch.Tensor):
    """(index, value) from packed keys on any device (CPU-side helper for tests/bench)."""
    k = keys.to(torch.int64)
    low = k & 0xFFFFFFFF
    index = 0xFFFFFFFF - low
    hi = (k >> 32) & 0xFFFFFFFF
    pos = (hi & 0x80000000) != 0
    bits = torch.where(pos, hi & 0x7FFFFFFF, (~hi) & 0xFFFFFFFF)
    value = bits.to(torch.int32).view(torch.float32)
    return index, value


def encode_host_keys(values: torch.Tensor, index: torch.Tensor) -> torch.Tensor:
    """Packed keys (int64 storage of the uint64 key) from per-frame max values and indices.

    Same packing as make_key in csrc/common.cuh: ordered float32 bits in the high word,
    0xFFFFFFFF - index in the low word.
    """
    v = values.to(torch.float32) + 0.0                     # -0.0 -> +0.0
    bits = v.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    neg = (bits & 0x80000000) != 0
    ordered = torch.where(neg, (~bits) & 0xFFFFFFFF, bits | 0x80000000)
    return (ordered << 32) | (0xFFFFFFFF - index.to(torch.int64))


def local_argmax_keys(z: torch.Tensor, row_offset: int = 0) -> torch.Tensor:
    """Keys of a (F, J_local) map block whose first column is global candidate `row_offset`."""
    vals, idx = z.max(dim=1)
    first = (z == vals[:, None]).to(torch.int8).argmax(dim=1)   # lowest index among ties
    return encode_host_keys(vals, first + row_offset)
