"""BASELINE config 5 (and the config 2 sweeps): complexity / throughput sweep.

    python tools/sweep_cfg5.py [--workload cfg5] [--quick] > gpurun_out/cfg5_sweep.jsonl

On the config-3 geometry (far-field UCA, J = 32760) this reports, one JSON line each:
  * batch sweep   F in 1 .. 65536 frames, SSPI (2JP) chain: maps/s (CUDA-graph replays,
                  L2 flushed between replays) and the map kernel's z-write GB/s;
  * nnz sweep     SSPI with q = 1 .. 32 kept entries per (candidate, pair) (global top-Q,
                  interpolation.py:155-175): maps/s, engine, parity vs the float64 oracle
                  of the same operator, and the map / localisation error vs the
                  conventional map (the reference's metrics.py:136-172 quantities);
  * rank sweep    SLRI with R = 1 .. 64: the same columns.
The conventional reference for the approximation errors is the GPU 3xTF32 map
(<= 5e-6 from float64, far below the approximation errors measured here).
With --workload cfg2 the sweeps are config 2's (rank {1..32}, nnz {1..16}).
"""

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2306_08514_b200 as s  # noqa: E402
from paper_2306_08514_b200 import maps, workloads  # noqa: E402
from paper_2306_08514_b200.pipeline import MapPipeline  # noqa: E402
from oracle import srp_oracle as O  # noqa: E402

FLUSH = None


def graph_ms(pipe, reps):
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    pipe.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        FLUSH.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pipe.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def loc_err(grid, i_est, i_ref):
    p = np.asarray(grid.points)
    if grid.mode == "ff":
        c = np.clip(np.sum(p[i_est] * p[i_ref], axis=1), -1.0, 1.0)
        return np.degrees(np.arccos(c))            # degrees
    return np.linalg.norm(p[i_est] - p[i_ref], axis=1)   # metres


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg5")
    ap.add_argument("--frames", type=int, default=4096)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    cfg2 = a.workload in ("cfg1", "cfg2")
    nnz_list = [1, 2, 4, 8, 16] if cfg2 else [1, 2, 4, 8, 16, 32]
    rank_list = [1, 2, 4, 8, 16, 32] if cfg2 else [1, 2, 4, 8, 16, 32, 64]
    batches = [1, 4, 16, 64, 256, 1024, 4096, 16384, 65536]
    if a.quick:
        batches = [1, 64, 1024, 16384]
        nnz_list, rank_list = nnz_list[:3], rank_list[::2]
    wl = workloads.make(a.workload, num_frames=max(batches + [a.frames]) if not cfg2 else a.frames)
    f_main = min(a.frames, wl.num_frames)
    x_dev = torch.from_numpy(wl.samples.astype(np.float32)).cuda()
    interp = s.build_interp_matrix(wl.tdoa, wl.spec, wl.frame, max_bytes=1 << 36)
    j, p_count = wl.grid.num_points, wl.pairs.num_pairs
    head = {"workload": a.workload, "J": j, "P": p_count, "S": wl.spec.total_samples,
            "frame_len": wl.frame.frame_len, "gpu": torch.cuda.get_device_name()}
    print(json.dumps({"sweep": "header", **head}), flush=True)

    def pipe_for(variant, op, frames, engine="auto"):
        pipe = MapPipeline(variant, op, wl.frame, wl.pairs, wl.spec, frames=frames, engine=engine)
        n = pipe.input.shape[1]
        pipe.input.copy_(x_dev[:, :n])
        return pipe

    # conventional reference maps (GPU 3xTF32) for the error columns, on nf_err frames
    nf_err = 64
    conv = s.steering_operator(wl.tdoa, wl.frame)
    g = s.gcc_frames(x_dev, wl.frame, wl.pairs, range(nf_err), tf32=False)
    z_conv, i_conv = s.srp_map_exact(conv, g, precision="tf32x3", argmax=True)
    z_conv = z_conv.cpu().numpy().astype(np.float64)
    i_conv = i_conv.cpu().numpy()
    # float64 oracle samples of the first 8 frames (parity of each operator)
    nf_or = 8
    xr = wl.samples[:, :(nf_or - 1) * wl.frame.hop + wl.frame.frame_len].astype(np.float64)
    win = O.frame_window(wl.frame.frame_len, wl.frame.window)
    psi = O.fd_gcc(O.stft_frames(xr, wl.frame.frame_len, wl.frame.hop, win, np.arange(nf_or)), wl.pairs.pairs)
    xi_ref = O.td_gcc_samples(psi, wl.spec.counts, wl.frame.half_len, "ifft")

    def errors(variant, op, pipe):
        pipe.run(x_dev[:, :pipe.input.shape[1]])
        torch.cuda.synchronize()
        z = pipe.z[:nf_err].cpu().numpy().astype(np.float64)
        idx = pipe.index[:nf_err].cpu().numpy()
        if variant == "sspi":
            z_or = O.sspi_map(op.values, op.col_indices, op.row_splits, xi_ref)
        else:
            z_or = O.slri_map(op.tall, op.fat, xi_ref)
        parity = float(O.normalized_max_error(z[:nf_or], z_or).max())
        eps = [O.map_error(z[f], z_conv[f]) for f in range(nf_err)]
        le = loc_err(wl.grid, idx, i_conv)
        return {"parity_max_err_vs_oracle": parity, "eps_z_db_mean": float(np.mean(eps)),
                "loc_err_mean": float(np.mean(le)), "loc_err_median": float(np.median(le)),
                "loc_err_unit": "deg" if wl.grid.mode == "ff" else "m",
                "argmax_eq_conv_frac": float(np.mean(idx == i_conv))}

    # ---- nnz sweep (SSPI) and rank sweep (SLRI) at f_main frames
    for q in nnz_list:
        t0 = time.perf_counter()
        sp = s.truncate_sparse(interp, min(interp.matrix.size,   # q > 2N_p+1 saturates at keep-all
                                           s.resolve_sparsity(f"{q}jp", j, p_count, interp.matrix.size)))
        fit_s = time.perf_counter() - t0
        pipe = pipe_for("sspi", sp, f_main)
        ms = graph_ms(pipe, 10)
        eng = "fused" if pipe.uses_fused_chain() else maps.map_engine("sspi", sp, "auto", f_main, bounded=True)
        row = {"sweep": "nnz", "nnz_per_cand_pair": q, "kept": int(sp.values.shape[0]), "frames": f_main,
               "ms_per_batch": ms, "maps_per_s": f_main / (ms / 1e3), "engine": eng,
               "host_fit_s": fit_s, **errors("sspi", sp, pipe)}
        print(json.dumps(row), flush=True)
        del pipe
    for r in rank_list:
        lr = s.truncate_low_rank(interp, r)
        pipe = pipe_for("slri", lr, f_main)
        ms = graph_ms(pipe, 10)
        row = {"sweep": "rank", "rank": r, "frames": f_main, "ms_per_batch": ms,
               "maps_per_s": f_main / (ms / 1e3), "engine": "fused" if pipe.uses_fused_chain() else "unfused",
               **errors("slri", lr, pipe)}
        print(json.dumps(row), flush=True)
        del pipe

    # ---- batch sweep (SSPI 2JP)
    if not cfg2:
        sp = s.truncate_sparse(interp, s.resolve_sparsity("2jp", j, p_count, interp.matrix.size))
        for fb in batches:
            if fb > wl.num_frames:
                continue
            for eng in ("tc", "tile", "tile_f16", "band", "auto"):
                pipe = pipe_for("sspi", sp, fb, eng)
                ms = graph_ms(pipe, 10 if fb >= 1024 else 30)
                row = {"sweep": "batch", "frames": fb, "ms_per_batch": ms, "maps_per_s": fb / (ms / 1e3),
                       "z_write_GBps": fb * j * 4 / (ms / 1e3) / 1e9, "engine": eng,
                       "auto_picks": maps.map_engine("sspi", sp, "auto", fb, bounded=True)}
                print(json.dumps(row), flush=True)
                del pipe
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
