for d in 0 1 2 3; do SRPGPU_CONV_DBG=$d timeout 90 python - <<'PY'
import os, torch, time
import paper_2306_08514_b200 as s
from paper_2306_08514_b200 import workloads
wl = workloads.make("cfg3", num_frames=4096)
x = torch.from_numpy(wl.samples).cuda()
op = s.steering_operator(wl.tdoa, wl.frame)
g = s.gcc_frames(x, wl.frame, wl.pairs, range(4096), tf32=True)
for _ in range(2): z = s.srp_map_exact(op, g)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5): z = s.srp_map_exact(op, g)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
print("dbg", os.environ["SRPGPU_CONV_DBG"], f"{ms:.3f} ms", f"{4*32760*28*255*4096/ms/1e9:.1f} TFLOPS")
PY
done
