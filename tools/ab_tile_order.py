"""A/B of the gathered-window engine's map output: straight into grid order vs tile order
+ untile pass (maps.TILE_GRID_ORDER), cfg4 geometry, with bit-equality of the two maps.

    python tools/ab_tile_order.py [--frames 10000] [--reps 5]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2306_08514_b200 as s  # noqa: E402
from paper_2306_08514_b200 import maps, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=10000)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--modes", default="tile,grid")
    a = ap.parse_args()
    wl = workloads.make("cfg4", num_frames=a.frames)
    op = s.sparse_interp_fixed(wl.tdoa, wl.spec, wl.frame, 2)
    x = torch.from_numpy(wl.samples).cuda()
    xi = s.frames_to_samples(x, wl.frame, wl.pairs, wl.spec, range(a.frames), planes=True, natural=True)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    out = {}
    modes = [m == "grid" for m in a.modes.split(",")]
    for mode in modes:
        maps.TILE_GRID_ORDER = mode
        z, idx = s.sspi_map(op, xi, argmax=True, engine="tile")
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            z, idx = s.sspi_map(op, xi, argmax=True, engine="tile")
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out["grid" if mode else "tile"] = {"ms": sorted(ts)[len(ts) // 2], "all": ts}
        out[f"z_{mode}"] = z.clone() if mode else z
        out[f"i_{mode}"] = idx.clone()
    if len(modes) == 2:
        same = bool(torch.equal(out.pop("z_True"), out.pop("z_False")) and torch.equal(out.pop("i_True"),
                                                                                       out.pop("i_False")))
        out["bit_identical"] = same
    for k in [k for k in out if k.startswith(("z_", "i_"))]:
        out.pop(k)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
