"""Multi-process (gloo, world_size 2) coverage of the frame- and candidate-partitioned paths.

On GPUs the same functions run over NCCL (bench.py under torchrun); the keys are
the 8-byte packed per-frame argmax keys of the map kernels.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_08514_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _maps(frames, cands, seed=0):
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((frames, cands)).astype(np.float32)
    z[3, [5, cands - 2]] = 50.0          # tie straddling the two candidate blocks
    z[4, :] = -1.0                        # all-equal row: lowest index wins
    z[5, 7] = -0.0
    z[5, :] = np.minimum(z[5, :], -0.5)
    z[5, 7] = 0.0
    return z


def _worker(rank, world, port, frames, cands, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z = torch.from_numpy(_maps(frames, cands))
    # frame partition: each rank maps its own frames, all-gather the keys
    f0, nf = D.partition(frames, world, rank)
    keys = D.local_argmax_keys(z[f0:f0 + nf])
    allk = D.gather_frame_keys(keys, frames)
    idx_f, val_f = D.decode_host_keys(allk)
    # candidate partition: each rank owns a block of candidates for all frames
    c0, nc = D.partition(cands, world, rank)
    ck = D.local_argmax_keys(z[:, c0:c0 + nc], row_offset=c0)
    red = D.reduce_candidate_keys(ck)
    idx_c, val_c = D.decode_host_keys(red)
    out[rank] = (idx_f.numpy(), val_f.numpy(), idx_c.numpy(), val_c.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("frames,cands", [(10, 37), (7, 64)])
def test_two_rank_partitions_match_single_process(frames, cands):
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    out = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, frames, cands, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    z = _maps(frames, cands)
    ref_idx = np.argmax(z, axis=1)           # np.argmax: first maximum (srp.py:74-80)
    for r in range(2):
        idx_f, val_f, idx_c, val_c = out[r]
        np.testing.assert_array_equal(idx_f, ref_idx)
        np.testing.assert_array_equal(idx_c, ref_idx)
        np.testing.assert_array_equal(val_f, z.max(axis=1))
        np.testing.assert_array_equal(val_c, z.max(axis=1))
    assert ref_idx[3] == 5 and ref_idx[4] == 0


def test_key_order_matches_argmax_rule():
    vals = torch.tensor([1.0, 1.0, -2.0, 3.0, -0.0, 0.0])
    idx = torch.tensor([9, 4, 1, 7, 2, 3])
    keys = D.encode_host_keys(vals, idx)
    order = torch.argsort(D.keys_to_signed(keys), descending=True)
    # largest value first; equal values -> lower index first; -0.0 ties +0.0
    assert idx[order].tolist() == [7, 4, 9, 2, 3, 1]
    i, v = D.decode_host_keys(keys)
    assert i.tolist() == idx.tolist()
    assert v.tolist() == [1.0, 1.0, -2.0, 3.0, 0.0, 0.0]


def _pipelined_worker(rank, world, port, frames, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    f0, nf = D.partition(frames * world, world, rank)
    seen = []
    slots = [torch.zeros(nf, dtype=torch.int64) for _ in range(3)]

    def step(k):
        def run():
            i = len(seen)
            slots[k].copy_(torch.arange(f0, f0 + nf, dtype=torch.int64) + 1000 * i)   # step i's result
            seen.append(i)
            return slots[k]
        return run

    outs = D.pipelined_steps([step(k) for k in range(3)], steps, frames * world)
    out[rank] = [o.numpy().copy() for o in outs]
    dist.barrier()
    dist.destroy_process_group()


def test_pipelined_gathers_two_ranks():
    """bench.py's N > 1 step loop: each step's per-frame results are all-gathered
    asynchronously; the two output buffers hold the last two steps of every rank."""
    frames, steps = 5, 7
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_pipelined_worker, args=(r, 2, port, frames, steps, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    base = np.arange(2 * frames)
    for r in range(2):
        last, prev = out[r][(steps - 1) % 2], out[r][(steps - 2) % 2]
        np.testing.assert_array_equal(last, base + 1000 * (steps - 1))
        np.testing.assert_array_equal(prev, base + 1000 * (steps - 2))


def test_pipelined_steps_single_process():
    calls = []
    outs = D.pipelined_steps([lambda: calls.append(1) or torch.zeros(3, dtype=torch.int64)], 4, 3)
    assert outs is None and len(calls) == 4
