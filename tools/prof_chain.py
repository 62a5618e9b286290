"""Run one workload's hot-path chain eagerly a few times (for ncu / compute-sanitizer).

    python tools/prof_chain.py --workload cfg2 --variant sspi --reps 3
"""

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2306_08514_b200 as s  # noqa: E402
from paper_2306_08514_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--variant", default="sspi")
    ap.add_argument("--frames", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--nnz", default="2jp")
    ap.add_argument("--rank", type=int, default=16)
    ap.add_argument("--engine", default="auto", help="sspi / si / slri / lr map engine")
    a = ap.parse_args()
    frames = a.frames or {"cfg1": 100, "cfg2": 1000, "cfg3": 10000, "cfg4": 10000}.get(a.workload, 1000)
    wl = workloads.make(a.workload, num_frames=frames)
    x = torch.from_numpy(wl.samples).cuda()
    rng = range(frames)
    if a.variant == "sspi" and a.workload == "cfg4":     # dense Lambda infeasible: fixed nnz per (i, p)
        from paper_2306_08514_b200 import maps
        op = s.sparse_interp_fixed(wl.tdoa, wl.spec, wl.frame, 2)
        eng = maps.map_engine("sspi", op, a.engine, frames)
        for _ in range(a.reps):
            xi = s.frames_to_samples(x, wl.frame, wl.pairs, wl.spec, rng, **s.maps.plane_args(eng))
            z, idx = s.sspi_map(op, xi, argmax=True, engine=eng)
    elif a.variant in ("sspi", "slri", "si"):
        interp = s.build_interp_matrix(wl.tdoa, wl.spec, wl.frame, max_bytes=1 << 36)
        if a.variant == "sspi":
            op = s.truncate_sparse(interp, s.resolve_sparsity(a.nnz, wl.grid.num_points,
                                                              wl.pairs.num_pairs, interp.matrix.size))
        elif a.variant == "slri":
            op = s.truncate_low_rank(interp, a.rank)
        else:
            op = interp
        from paper_2306_08514_b200 import maps
        if a.engine == "fused":          # frontend + map + argmax in one kernel
            chain = maps.frames_to_slri_map if a.variant == "slri" else maps.frames_to_sspi_map
            for _ in range(a.reps):
                z, idx = chain(op, x, wl.frame, wl.pairs, wl.spec, rng)
            torch.cuda.synchronize()
            return
        fn = {"sspi": s.sspi_map, "slri": s.slri_map, "si": s.si_map}[a.variant]
        eng = maps.map_engine(a.variant, op, a.engine, frames)
        for _ in range(a.reps):
            xi = s.frames_to_samples(x, wl.frame, wl.pairs, wl.spec, rng, **s.maps.plane_args(eng))
            z, idx = fn(op, xi, argmax=True, engine=a.engine)
    elif a.variant == "conv":          # on-chip steering (bench variant "conv")
        op = s.steering_operator(wl.tdoa, wl.frame)
        for _ in range(a.reps):
            g = s.gcc_frames(x, wl.frame, wl.pairs, rng, tf32=True)
            z, idx = s.srp_map_exact(op, g, argmax=True)
    else:                              # stored operator: conv_h (SrpMatrix) or lr
        srp = s.build_srp_matrix(wl.tdoa, wl.frame, max_bytes=1 << 36)
        op = srp if a.variant == "conv_h" else s.truncate_srp_matrix(srp, a.rank)
        for _ in range(a.reps):
            g = s.gcc_frames(x, wl.frame, wl.pairs, rng, tf32=(a.variant == "conv_h"))
            z, idx = (s.srp_map_exact(op, g, argmax=True) if a.variant == "conv_h"
                      else s.lr_map(op, g, argmax=True, engine=a.engine))
    torch.cuda.synchronize()
    print("ok", a.workload, a.variant, frames, int(idx[0]))


if __name__ == "__main__":
    main()
