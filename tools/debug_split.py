import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2306_08514_b200 as s
from paper_2306_08514_b200 import _native as nat, _device as dev, maps
from conftest import load_golden, scene_objects
from oracle import srp_oracle as O

g = load_golden("cfg3_small")
array, pairs, grid, frame, tdoa, spec = scene_objects(g)
op = s.steering_operator(tdoa, frame)
psi = torch.from_numpy(g["psi"].astype(np.complex64)).cuda()
F = psi.shape[0]; n = op.num_pairs * op.num_bins; ld = (2 * n + 3) // 4 * 4
v = torch.view_as_real(psi).reshape(F, 2 * n).contiguous()
xt = maps._xtab_device(op)
def run(vp, split):
    z = torch.empty((F, op.num_candidates), device="cuda")
    nat.call("srpgpu_srp_map_tdoa", dev.ptr(vp), ld, F, op.num_pairs, op.num_bins + 1, dev.ptr(xt),
             op.num_candidates, split, dev.ptr(z), None, dev.stream_ptr())
    torch.cuda.synchronize()
    return z.cpu().numpy()
vp = torch.zeros((2 * F, ld), device="cuda")
nat.call("srpgpu_split_tf32", dev.ptr(v), 2 * n, dev.ptr(vp), ld, F, 2 * n, dev.stream_ptr())
torch.cuda.synchronize()
hi, lo = vp[:F].cpu().numpy(), vp[F:].cpu().numpy()
print("lo nonzero frac", np.mean(lo[:, :2 * n] != 0), "max |lo|", np.abs(lo).max(), "hi-v err", np.abs(hi[:, :2*n] + lo[:, :2*n] - v.cpu().numpy()).max())
zref = g["z_conv"]
z1 = run(vp, 0)
z3 = run(vp, 1)
vp0 = vp.clone(); vp0[F:] = 0
z3b = run(vp0, 1)
print("tf32 err", O.normalized_max_error(z1, zref).max())
print("3xtf32 err", O.normalized_max_error(z3, zref).max())
print("3x with lo_B=0 err", O.normalized_max_error(z3b, zref).max(), "diff vs 3x", np.abs(z3 - z3b).max())
srp = s.build_srp_matrix(tdoa, frame)
zf = s.srp_map_exact(srp, s.FdGcc(psi, pairs.num_pairs, frame.num_bins, "phat"), precision="fp32").cpu().numpy()
print("fp32 simt err", O.normalized_max_error(zf, zref).max())

# (1) B_lo := B_hi  ->  (2 A_hi + A_lo) B_hi ~= 2 z
vp2 = vp.clone(); vp2[F:] = vp2[:F]
z_dbl = run(vp2, 1)
print("B_lo=B_hi: max |z_split - 2 z_tf32| / max|z|", np.abs(z_dbl - 2 * z1).max() / np.abs(z1).max())
# (2) B_lo := 0 -> (A_hi + A_lo) B_hi vs exact H . psi_hi (float64)
psi_hi = (hi[:, 0:2 * n:2] + 1j * hi[:, 1:2 * n:2]).astype(np.complex128)
zref_hi = O.srp_map_exact(srp.matrix, psi_hi)
print("B_lo=0 vs f64 H . psi_hi:", O.normalized_max_error(z3b, zref_hi).max(),
      " tf32 vs same:", O.normalized_max_error(z1, zref_hi).max())

def rna_tf32(x):
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x1000) & 0xFFFFE000     # round half away (magnitude) on the 13 dropped bits
    return u.astype(np.uint32).view(np.float32)
A = np.empty((srp.matrix.shape[0], 2 * n), dtype=np.float32)
A[:, 0::2] = srp.matrix.real; A[:, 1::2] = -srp.matrix.imag
Ahi = rna_tf32(A); Alo = rna_tf32(A - Ahi)
Bhi, Blo = hi[:, :2 * n].astype(np.float64), lo[:, :2 * n].astype(np.float64)
Ahi64, Alo64 = Ahi.astype(np.float64), Alo.astype(np.float64)
z_emul3 = 2 * (Bhi @ Ahi64.T + Blo @ Ahi64.T + Bhi @ Alo64.T)
z_emul1 = 2 * (Bhi @ Ahi64.T)
z_emulA = 2 * (Bhi @ (Ahi64 + Alo64).T)
print("emul 3x err vs ref", O.normalized_max_error(z_emul3, zref).max(), " gpu3x vs emul3x", O.normalized_max_error(z3, z_emul3).max())
print("emul tf32 vs gpu tf32", O.normalized_max_error(z1, z_emul1).max())
print("emul (Ahi+Alo)Bhi vs gpu B_lo=0", O.normalized_max_error(z3b, z_emulA).max())

# stored-H path: operands known exactly on the host (RNE-rounded H and psi)
from paper_2306_08514_b200.maps import _tf32_rne_host, steering_device
h2 = steering_device(srp, tf32=True)[:, :2 * n].cpu().numpy().astype(np.float64)
gcc_r = s.gcc_frames  # unused
vr = torch.empty((F, ld), device="cuda")
nat.call("srpgpu_round_tf32", dev.ptr(v), 2 * n, dev.ptr(vr), ld, F, 2 * n, dev.stream_ptr())
zs_ = s.srp_map_exact(srp, s.FdGcc(psi, pairs.num_pairs, frame.num_bins, "phat")).cpu().numpy()
Br = vr[:, :2 * n].cpu().numpy().astype(np.float64)
z_emul_s = 2 * (Br @ h2.T)
print("stored-H: gpu vs exact emulation of its own operands", O.normalized_max_error(zs_, z_emul_s).max(),
      " emul vs ref", O.normalized_max_error(z_emul_s, zref).max())
# accumulation-length dependence: only the first pair (K' = 2B) of the operands
p1 = 2 * op.num_bins
z_p1 = 2 * (Br[:, :p1] @ h2[:, :p1].T)
