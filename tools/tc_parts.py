"""Time the tensor-core interpolation kernel with z only, argmax only, and both (CUDA graphs)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_08514_b200 as s  # noqa: E402
from paper_2306_08514_b200 import workloads, maps, _native as nat  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
wl = workloads.make(cfg)
f = wl.num_frames
x = torch.from_numpy(wl.samples.astype(np.float32)).cuda()
xi = s.frames_to_samples(x, wl.frame, wl.pairs, wl.spec, range(f), planes=True)
interp = s.build_interp_matrix(wl.tdoa, wl.spec, wl.frame, max_bytes=1 << 36)
sp = s.truncate_sparse(interp, s.resolve_sparsity("2jp", wl.grid.num_points, wl.pairs.num_pairs, interp.matrix.size))
op = maps.dense_from_sparse(sp)
z = torch.empty((f, op.num_rows), device="cuda")
k = torch.empty(f, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
out = {"cfg": cfg}
for name, zp, kp in (("z+keys", z.data_ptr(), k.data_ptr()), ("z", z.data_ptr(), 0), ("keys", 0, k.data_ptr())):
    call = lambda: nat.call("srpgpu_interp_map_tc", xi.bf16_planes.data_ptr(), f, op.planes.data_ptr(), op.num_rows,
                            op.cols8, zp, kp, torch.cuda.current_stream().cuda_stream)
    call(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        call()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    out[name] = float(np.median(ts))
print(json.dumps(out))
