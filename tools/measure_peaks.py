"""Measure the TF32 tensor (cuBLAS) and FP32 SIMT peaks on this B200, the way
MEASURED_PEAKS.json measures bf16: 8192^3 GEMM, best of 10, CUDA events.
Writes profiles/measured_peaks_extra.json (used as the TF32 / FP32 roofline denominators)."""

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gemm_tflops(dtype, tf32: bool, n=8192, reps=10):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2.0 * n ** 3 / (best / 1e3) / 1e12


def main():
    props = torch.cuda.get_device_properties(0)
    out = {
        "gpu": props.name,
        "tf32_tflops": gemm_tflops(torch.float32, True),
        "fp32_tflops": gemm_tflops(torch.float32, False),
        "bf16_tflops": gemm_tflops(torch.bfloat16, False),
        "how": "torch.matmul 8192^3, best of 10, CUDA events; tf32 = allow_tf32 (cuBLAS TF32 tensor cores), "
               "fp32 = allow_tf32 off (cuBLAS FP32 SIMT)",
    }
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "measured_peaks_extra.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
