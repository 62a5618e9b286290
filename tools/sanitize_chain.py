"""Small end-to-end run of every kernel family (for compute-sanitizer memcheck)."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2306_08514_b200 as s  # noqa: E402
from paper_2306_08514_b200 import workloads  # noqa: E402


def main():
    wl = workloads.make("cfg1", num_frames=70)
    x = torch.from_numpy(wl.samples).cuda()
    xi = s.frames_to_samples(x, wl.frame, wl.pairs, wl.spec)
    interp = s.build_interp_matrix(wl.tdoa, wl.spec, wl.frame)
    sp = s.truncate_sparse(interp, 2 * wl.grid.num_points * wl.pairs.num_pairs)
    z1, i1 = s.sspi_map(sp, xi, argmax=True)
    z1b = s.sspi_map(sp, s.TdGccSamples(xi.values[:5].contiguous(), wl.spec))     # rows kernel
    z2 = s.si_map(interp, xi)
    lr = s.truncate_low_rank(interp, 8)
    z3, i3 = s.slri_map(lr, xi, argmax=True)
    gcc = s.gcc_frames(x, wl.frame, wl.pairs, tf32=True)
    z4, i4 = s.srp_map_exact(s.steering_operator(wl.tdoa, wl.frame), gcc, argmax=True)
    srp = s.build_srp_matrix(wl.tdoa, wl.frame)
    z5, i5 = s.srp_map_exact(srp, gcc, argmax=True)
    z6 = s.srp_map_exact(srp, gcc, precision="fp32")
    lrs = s.truncate_srp_matrix(srp, 4)
    z7 = s.lr_map(lrs, s.gcc_frames(x, wl.frame, wl.pairs))
    y = s.stft_frame(x, wl.frame, range(0, 10))
    g2 = s.fd_gcc(y, wl.pairs)
    xi2 = s.td_gcc_samples(g2, wl.spec)
    xi3 = s.spectra_to_samples(y, wl.pairs, wl.spec)
    loc = s.locate(z1[0], wl.grid)
    torch.cuda.synchronize()
    print("ok", int(i1[0]), int(i3[0]), int(i4[0]), int(i5[0]), float(z6[0, 0]), float(z7[0, 0]), loc[0],
          xi2.values.shape, xi3.values.shape, z1b.shape, z2.shape)


if __name__ == "__main__":
    main()
