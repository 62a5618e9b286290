"""Time the frontend kernels (warp per frame / warp per task / block) on each workload.

    python tools/bench_frontend.py [--workloads cfg1,cfg2,cfg3,cfg4] [--reps 50]

Each measurement is a CUDA graph of one `frames_to_samples` launch (the layout the
workload's map engine reads), timed with CUDA events over `reps` replays after warm-up,
L2 flushed between replays.  Prints one JSON line per (workload, frames, kernel).
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2306_08514_b200 as s  # noqa: E402
from paper_2306_08514_b200 import workloads  # noqa: E402
from paper_2306_08514_b200.frontend import frontend_kernel  # noqa: E402

DEFAULT_FRAMES = {"cfg1": 100, "cfg2": 1000, "cfg3": 10000, "cfg4": 10000}
ENGINE = {"cfg1": "band", "cfg2": "band", "cfg3": "tile", "cfg4": "tile"}   # the map engine whose planes are written


def time_graph(fn, reps, flush):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="cfg1,cfg2,cfg3,cfg4")
    ap.add_argument("--frames", default="", help="comma list overriding the workload's frame count")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--kernels", default="warp,task,block")
    ap.add_argument("--rounds", type=int, default=1, help="alternate the kernels this many times (median)")
    a = ap.parse_args()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for name in a.workloads.split(","):
        frame_list = [int(f) for f in a.frames.split(",")] if a.frames else [DEFAULT_FRAMES[name]]
        wl = workloads.make(name, num_frames=max(frame_list))
        x = torch.from_numpy(wl.samples).cuda()
        pa = s.maps.plane_args(ENGINE.get(name, "band"))
        for frames in frame_list:
            times = {k: [] for k in a.kernels.split(",")}
            for _ in range(a.rounds):
                for k in times:
                    with frontend_kernel(k):
                        try:
                            times[k].append(time_graph(
                                lambda: s.frames_to_samples(x, wl.frame, wl.pairs, wl.spec, range(frames), **pa),
                                a.reps, flush))
                        except Exception as exc:  # noqa: BLE001
                            times[k].append(float("nan"))
                            print(json.dumps({"workload": name, "frames": frames, "kernel": k, "error": str(exc)}))
            for k, ts in times.items():
                ms = sorted(ts)[len(ts) // 2]
                print(json.dumps({"workload": name, "frames": frames, "kernel": k, "planes": pa, "ms": ms, "ns_per_frame": ms * 1e6 / frames,
                                  "all_ms": ts}), flush=True)

if __name__ == "__main__":
    main()
