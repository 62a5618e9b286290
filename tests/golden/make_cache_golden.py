"""SRPM cache fixtures written by the reference itself (SURVEY §8(f) #3 parity pins).

Run in the build container (where /root/reference exists):

    python tests/golden/make_cache_golden.py

For a small near-field scene this builds every operator kind (conv, lr, si, slri,
sspi) with the reference builders exactly as `cli.build_operator` does
(cli.py:75-130), writes it with the reference `save_cache` and the reference
`params_hash` digest (cli.py:46-66, fed a minimal stand-in for RunConfig), and
records the reference maps `cli.evaluate_map` computes from the operator it reads
back (`load_cache` + `operator_from_bundle`, cli.py:133-159) for a few frames.
Outputs: tests/golden/cache/<kind>.srpm and tests/golden/cache_golden.npz.
"""

from __future__ import annotations

import os
import sys
from types import SimpleNamespace

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from srpmap import (FrameSpec, MicrophoneArray, build_interp_matrix, build_nf_grid,  # noqa: E402
                    build_srp_matrix, enumerate_pairs, fd_gcc, sample_spec, stft_frame,
                    tdoa_table, truncate_low_rank, truncate_sparse, truncate_srp_matrix)
from srpmap import cli  # noqa: E402
from srpmap.cache import load_cache, save_cache  # noqa: E402
from srpmap.config import MethodSpec  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "cache")


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(20306)
    positions = np.array([[0.30, 0.32, 0.0], [0.42, 0.28, 0.0], [0.35, 0.45, 0.0], [0.27, 0.40, 0.0]])
    array = MicrophoneArray(positions, 343.0)
    grid = build_nf_grid((0.0, 0.0, 0.0), (0.7, 0.7, 0.0), 0.1)
    frame = FrameSpec(frame_len=128, sample_rate=16000.0)
    room = np.array([4.0, 4.0, 3.0])
    cfg = SimpleNamespace(scenario=SimpleNamespace(mode="nf", room=room, array=array, grid=grid),
                          frame=frame, weighting="phat", n_aux=2)
    pairs = enumerate_pairs(array)
    tdoa = tdoa_table(array, pairs, grid)
    spec = sample_spec(tdoa, frame, cfg.n_aux)
    j, p, b = grid.num_points, pairs.num_pairs, frame.num_bins

    nf = 3
    n = (nf - 1) * frame.hop + frame.frame_len
    samples = 0.3 * rng.standard_normal((array.num_mics, n))
    common = rng.standard_normal(n + 8)          # a common source with per-channel delays: peaked maps
    for ch, d in enumerate(rng.integers(0, 4, array.num_mics)):
        samples[ch] += common[d:d + n]
    gccs = [fd_gcc(stft_frame(samples, frame, f), pairs) for f in range(nf)]

    meta0 = {"num_pairs": p, "num_bins": b, "num_candidates": j, "half_len": frame.half_len,
             "n_aux": cfg.n_aux, "path": "ifft"}
    interp = build_interp_matrix(tdoa, spec, frame)
    srp = build_srp_matrix(tdoa, frame)
    lr = truncate_srp_matrix(srp, 4)
    slri = truncate_low_rank(interp, 4)
    keep = 2 * j * p
    sp = truncate_sparse(interp, keep)
    builds = {
        "conv": ({"matrix": srp.matrix}, {}, None, None),
        "lr": ({"tall": lr.tall, "fat": lr.fat, "singular_values": lr.singular_values}, {"rank": 4}, 4, None),
        "si": ({"matrix": interp.matrix, "counts": spec.counts}, {}, None, None),
        "slri": ({"tall": slri.tall, "fat": slri.fat, "singular_values": slri.singular_values,
                  "counts": spec.counts}, {"rank": 4}, 4, None),
        "sspi": ({"values": sp.values, "col_indices": sp.col_indices, "row_splits": sp.row_splits,
                  "counts": spec.counts}, {"keep": keep, "num_cols": sp.num_cols}, None, keep),
    }
    golden = {"positions": positions, "room": room, "speed_of_sound": np.float64(343.0),
              "grid_axes_x": grid.axes[0], "grid_axes_y": grid.axes[1], "grid_axes_z": grid.axes[2],
              "frame_len": np.int64(frame.frame_len), "sample_rate": np.float64(frame.sample_rate),
              "hop": np.int64(frame.hop), "n_aux": np.int64(cfg.n_aux), "samples": samples}
    for kind, (arrays, extra, rank, kp) in builds.items():
        meta = dict(meta0, **extra)
        method = MethodSpec(name=kind, rank=None if rank is None else str(rank),
                            sparsity=None if kp is None else str(kp), path="ifft")
        digest = cli.params_hash(cfg, method, rank=meta.get("rank"), keep=meta.get("keep"))
        path = os.path.join(OUT, f"{kind}.srpm")
        save_cache(path, kind, arrays, meta, digest)
        bundle = load_cache(path)
        op, sspec = cli.operator_from_bundle(bundle)
        z = np.stack([cli.evaluate_map(kind, op, sspec, frame, g, "ifft") for g in gccs])
        golden[f"{kind}_digest"] = np.array(digest)
        golden[f"{kind}_z"] = z
        print(f"{kind}: {os.path.getsize(path)} bytes, digest {digest[:12]}")
    np.savez_compressed(os.path.join(HERE, "cache_golden.npz"), **golden)


if __name__ == "__main__":
    main()
