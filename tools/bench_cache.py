"""Time SRPM cache -> device operator for the cfg3 conventional map (3.7 GB complex128).

    python tools/bench_cache.py [--dir /tmp]

Arms (same file, already in the page cache after a warm read):
  device : load_operator -> memory-mapped float64 blocks, H2D, srpgpu_c128_to_steering
  host   : the host conversion conj -> complex64 -> TF32 (RNE) in NumPy, then H2D
Prints one JSON line.
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2306_08514_b200 as s  # noqa: E402
from paper_2306_08514_b200 import maps, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", default="/tmp")
    ap.add_argument("--workload", default="cfg3")
    a = ap.parse_args()
    wl = workloads.make(a.workload, num_frames=8)
    srp = s.build_srp_matrix(wl.tdoa, wl.frame, max_bytes=1 << 36)
    path = os.path.join(a.dir, f"{a.workload}_conv.srpm")
    meta = {"num_pairs": wl.pairs.num_pairs, "num_bins": wl.frame.num_bins,
            "num_candidates": wl.grid.num_points, "half_len": wl.frame.half_len, "n_aux": 2, "path": "ifft"}
    s.save_cache(path, "conv", {"matrix": srp.matrix}, meta, "bench")
    nbytes = os.path.getsize(path)
    del srp
    with open(path, "rb") as fh:                      # warm the page cache for both arms
        while fh.read(1 << 28):
            pass

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    kind, op, _ = s.load_operator(path)
    h2 = maps.steering_device(op, tf32=True)
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0

    t0 = time.perf_counter()
    b = s.load_cache(path, mmap=False)
    h = b.arrays["matrix"]
    j, n = h.shape
    out = torch.zeros((j, (2 * n + 3) // 4 * 4), dtype=torch.float32, device="cuda")
    step = max(1, (256 << 20) // (16 * n))
    for r0 in range(0, j, step):
        blk = maps._tf32_rne_host(np.conj(h[r0:r0 + step]).astype(np.complex64).view(np.float32))
        out[r0:r0 + blk.shape[0], :2 * n] = torch.from_numpy(blk).cuda()
    torch.cuda.synchronize()
    t_host = time.perf_counter() - t0
    same = bool(torch.equal(out, h2))
    os.remove(path)
    print(json.dumps({"workload": a.workload, "file_bytes": nbytes, "device_s": t_dev, "host_s": t_host,
                      "device_gbs": nbytes / t_dev / 1e9, "host_gbs": nbytes / t_host / 1e9,
                      "speedup": t_host / t_dev, "bit_identical": same}))


if __name__ == "__main__":
    main()
