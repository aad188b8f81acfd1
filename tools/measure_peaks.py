#!/usr/bin/env python
"""Measure the compute peaks the sweep roofline needs:
FP64 (DGEMM), FP32 SIMT (SGEMM with TF32 off) and TF32 tensor-core (SGEMM
with TF32 on) throughput of this B200, via cuBLAS through torch.matmul
(library GEMMs are the reference ceiling, not the product path).  HBM
bandwidth comes from the driver-written MEASURED_PEAKS.json.

    python tools/measure_peaks.py > profiles/compute_peaks.json

Best of `reps` timed launches (CUDA events), N^3 GEMMs, 2 N^3 flops each.
"""
import json
import sys

import torch


def best_tflops(dtype, n, tf32, reps=8):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = float("inf")
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(reps):
        s.record()
        torch.matmul(a, b)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return 2.0 * n ** 3 / (best / 1e3) / 1e12


def main():
    dev = torch.cuda.get_device_properties(0)
    out = {
        "gpu": dev.name,
        "sm_count": dev.multi_processor_count,
        "fp64_tflops": round(best_tflops(torch.float64, 8192, False), 2),
        "fp32_simt_tflops": round(best_tflops(torch.float32, 8192, False), 2),
        "tf32_tensor_tflops": round(best_tflops(torch.float32, 8192, True), 2),
        "how": "cuBLAS via torch.matmul, 8192^3, best of 8 launches timed with CUDA events; "
               "tf32 = fp32 inputs with allow_tf32 (tensor cores), fp32_simt = allow_tf32 off",
        "torch": torch.__version__,
    }
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
