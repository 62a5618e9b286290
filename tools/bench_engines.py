"""Time the SSPI/SI map engines (tensor-core dense vs FP32 tiled band) on a workload.

    python tools/bench_engines.py [cfg3] [frames] [nnz tokens...]
Prints one JSON line per (token, engine): ms per map launch (CUDA events, L2 not
flushed: the map kernel's own operands are L2-resident in steady state), the split
kernel's share, and the normalized error of 8 frames against the float64 oracle.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2306_08514_b200 as s  # noqa: E402
from paper_2306_08514_b200 import workloads, maps  # noqa: E402
from oracle import srp_oracle as O  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    tokens = sys.argv[3:] or ["2jp"]
    wl = workloads.make(cfg, num_frames=frames or None)
    f = wl.num_frames
    x = torch.from_numpy(wl.samples.astype(np.float32)).cuda()
    xi = s.frames_to_samples(x, wl.frame, wl.pairs, wl.spec, range(f))
    interp = s.build_interp_matrix(wl.tdoa, wl.spec, wl.frame, max_bytes=1 << 36)
    nf = 8
    xr = wl.samples[:, :(nf - 1) * wl.frame.hop + wl.frame.frame_len].astype(np.float64)
    win = O.frame_window(wl.frame.frame_len, wl.frame.window)
    psi = O.fd_gcc(O.stft_frames(xr, wl.frame.frame_len, wl.frame.hop, win, np.arange(nf)), wl.pairs.pairs)
    xi_ref = O.td_gcc_samples(psi, wl.spec.counts, wl.frame.half_len, "ifft")
    for tok in tokens:
        keep = s.resolve_sparsity(tok, wl.grid.num_points, wl.pairs.num_pairs, interp.matrix.size)
        sp = s.truncate_sparse(interp, keep)
        z_ref = O.sspi_map(sp.values, sp.col_indices, sp.row_splits, xi_ref)
        for eng in ("tc", "band"):
            out = {}
            fn = lambda: s.sspi_map(sp, xi, argmax=True, engine=eng)
            z, idx = fn()
            torch.cuda.synchronize()
            out["ms"] = timed(fn)
            if eng == "tc":
                op = maps.dense_from_sparse(sp)
                planes, _, _ = maps.sample_planes(xi, op.num_cols)
                zz = torch.empty((f, op.num_rows), device="cuda")
                kk = torch.empty(f, dtype=torch.int64, device="cuda")
                out["ms_split"] = timed(lambda: maps.sample_planes(xi, op.num_cols))
                out["ms_kernel"] = timed(lambda: s._native.call(
                    "srpgpu_interp_map_tc", planes.data_ptr(), f, op.planes.data_ptr(), op.num_rows, op.cols8,
                    zz.data_ptr(), kk.data_ptr(), torch.cuda.current_stream().cuda_stream))
                out["cols8"] = op.cols8
            err = O.normalized_max_error(z[:nf].cpu().numpy(), z_ref)
            ok = O.peak_margin(z_ref) > 1e-4
            out.update({"cfg": cfg, "frames": f, "J": wl.grid.num_points, "S": wl.spec.total_samples,
                        "nnz": tok, "engine": eng, "max_err": float(err.max()),
                        "argmax_ok": bool(np.array_equal(idx[:nf].cpu().numpy()[ok], np.argmax(z_ref, 1)[ok])),
                        "zbytes_GBps": f * wl.grid.num_points * 4 / (out.get("ms_kernel", out["ms"]) * 1e6)})
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
