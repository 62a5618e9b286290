"""Time the batched `map` command end to end at cfg3 scale (recording file -> CSV).

    python tools/bench_batch.py [--frames 20000] [--dir /tmp]

Writes a float32 WAV of the cfg3 scene and an SSPI (2jp) SRPM cache, then times
`batch.cmd_map` (cache load + upload, WAV read, all frames mapped in batched CUDA
graphs, summary CSV) and, separately, `map_recording` alone.  One JSON line.
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch
from scipy.io import wavfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2306_08514_b200 as s  # noqa: E402
from paper_2306_08514_b200 import batch as B, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=20000)
    ap.add_argument("--dir", default="/tmp")
    ap.add_argument("--workload", default="cfg3")
    a = ap.parse_args()
    wl = workloads.make(a.workload, num_frames=a.frames)
    scene = B.RunScene(mode=wl.grid.mode, room=np.array([4.0, 4.0, 3.0]), array=wl.array, grid=wl.grid,
                       frame=wl.frame, weighting="phat", n_aux=2)
    interp = s.build_interp_matrix(wl.tdoa, wl.spec, wl.frame, max_bytes=1 << 36)
    keep = 2 * wl.grid.num_points * wl.pairs.num_pairs
    sp = s.truncate_sparse(interp, keep)
    meta = {"num_pairs": wl.pairs.num_pairs, "num_bins": wl.frame.num_bins, "num_candidates": wl.grid.num_points,
            "half_len": wl.frame.half_len, "n_aux": 2, "path": "ifft", "keep": keep, "num_cols": sp.num_cols}
    cache = os.path.join(a.dir, "bench_sspi.srpm")
    s.save_cache(cache, "sspi", {"values": sp.values, "col_indices": sp.col_indices, "row_splits": sp.row_splits,
                                 "counts": wl.spec.counts}, meta, B.scene_hash(scene, "sspi", meta))
    wav = os.path.join(a.dir, "bench_scene.wav")
    wavfile.write(wav, int(wl.frame.sample_rate), wl.samples.T.astype(np.float32))
    out = os.path.join(a.dir, "bench_map.csv")

    B.cmd_map(scene, cache, wav, out)                       # warm (first CUDA graphs, page cache)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = B.cmd_map(scene, cache, wav, out)
    torch.cuda.synchronize()
    t_cmd = time.perf_counter() - t0

    kind, op, spec = s.load_operator(cache)
    x, _ = B.load_audio(wav)
    B.map_recording(kind, op, spec, wl.frame, wl.pairs, x)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    B.map_recording(kind, op, spec, wl.frame, wl.pairs, x)
    torch.cuda.synchronize()
    t_map = time.perf_counter() - t0
    f = int(res.index.shape[0])
    for p in (cache, wav, out):
        os.remove(p)
    print(json.dumps({"workload": a.workload, "frames": f, "candidates": wl.grid.num_points,
                      "cmd_map_s": t_cmd, "cmd_map_frames_per_s": f / t_cmd,
                      "map_recording_s": t_map, "map_recording_frames_per_s": f / t_map,
                      "note": "cmd_map = cache load + upload + WAV read + maps + summary CSV"}))


if __name__ == "__main__":
    main()
