"""A/B of the gathered-window SSPI engines (fp16x3 "tile_f16" vs 3xTF32 "tile" vs bf16x3 "tile_bf16") at cfg4:
device time of the frontend and of the map per 10^4 frames, and parity against the
float64 oracle on a few frames.  Usage: python tools/bench_tile.py [--fit fixed|global]"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_08514_b200 as s  # noqa: E402
from paper_2306_08514_b200 import workloads  # noqa: E402
from oracle import srp_oracle as O  # noqa: E402


def timeit(fn, reps=5):
    flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fit", default="fixed")
    ap.add_argument("--frames", type=int, default=10000)
    ap.add_argument("--engines", default="tile_f16,tile,tile_bf16")
    ap.add_argument("--workload", default="cfg4")
    args = ap.parse_args()
    t0 = time.time()
    wl = workloads.make(args.workload, num_frames=args.frames)
    if args.fit == "fixed":
        sp = s.sparse_interp_fixed(wl.tdoa, wl.spec, wl.frame, 2)
    else:
        keep = s.resolve_sparsity("2jp", wl.grid.num_points, wl.pairs.num_pairs,
                                  wl.grid.num_points * wl.spec.total_samples)
        sp = s.truncate_sparse_streamed(wl.tdoa, wl.spec, wl.frame, keep)
    print(f"setup {time.time() - t0:.1f} s", flush=True)
    x = torch.from_numpy(wl.samples).cuda()
    nf = 4
    xi_ref = O.td_gcc_samples(O.fd_gcc(O.stft_frames(wl.samples[:, :(nf - 1) * wl.frame.hop + wl.frame.frame_len]
                                                     .astype(np.float64), wl.frame.frame_len, wl.frame.hop,
                                                     O.frame_window(wl.frame.frame_len, wl.frame.window),
                                                     np.arange(nf)), wl.pairs.pairs),
                              wl.spec.counts, wl.frame.half_len)
    if hasattr(sp, "kept"):
        z_ref = np.zeros((nf, wl.grid.num_points))
        for p in range(wl.pairs.num_pairs):
            k = int(sp.kept[p])
            z_ref += np.einsum("jk,fjk->fj", sp.values[p, :, :k], xi_ref[:, sp.cols[p, :, :k]])
    else:
        z_ref = O.sspi_map(sp.values, sp.col_indices, sp.row_splits, xi_ref)
    out = {}
    for eng in args.engines.split(","):
        t1 = time.time()
        pa = s.maps.plane_args(eng)
        xi = s.frames_to_samples(x, wl.frame, wl.pairs, wl.spec, range(args.frames), **pa)
        z, idx = s.sspi_map(sp, xi, argmax=True, engine=eng)
        torch.cuda.synchronize()
        setup = time.time() - t1
        err = O.normalized_max_error(z[:nf].cpu().numpy(), z_ref)
        ok = O.peak_margin(z_ref) > 1e-4
        agree = bool(np.array_equal(idx[:nf].cpu().numpy()[ok], np.argmax(z_ref, axis=1)[ok]))
        t_front = timeit(lambda: s.frames_to_samples(x, wl.frame, wl.pairs, wl.spec, range(args.frames), **pa))
        t_map = timeit(lambda: s.sspi_map(sp, xi, argmax=True, engine=eng))
        t_keys = timeit(lambda: s.sspi_map(sp, xi, argmax=True, out_map=False, engine=eng))
        op = s.maps.tile_from_sparse(sp, s.maps.spec_offsets(wl.spec), fmt=s.maps.TILE_ENGINES[eng]) \
            if eng in s.maps.TILE_ENGINES else None
        r = {"engine": eng, "frontend_ms": t_front, "map_ms": t_map, "map_argmax_only_ms": t_keys,
             "maps_per_s": args.frames / ((t_front + t_map) / 1e3), "err": float(err.max()), "argmax_agree": agree,
             "setup_s": setup}
        if op is not None:
            mma = 3 * 2.0 * op.num_tiles * 256 * op.mean_k * args.frames
            r.update({"mean_k": op.mean_k, "tiles": op.num_tiles,
                      "mma_tflops": mma / (t_keys / 1e3) / 1e12})
        print(json.dumps(r), flush=True)
        out[eng] = r
        del xi, z, idx


if __name__ == "__main__":
    main()
