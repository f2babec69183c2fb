"""Measured dense TF32 tensor-core throughput on this GPU (cuBLAS via
torch.matmul on FP32 inputs with TF32 allowed, 8192^3, best of 10 and back to
back for ~3 s), the denominator of bench.py's tensor bound (--tf32-tflops)."""
import json
import time

import torch


def main():
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    t0 = time.perf_counter()
    k = 0
    while time.perf_counter() - t0 < 3.0:
        for _ in range(20):
            a @ b
        torch.cuda.synchronize()
        k += 20
    sus = 2 * n ** 3 * k / (time.perf_counter() - t0) / 1e12
    print(json.dumps({"tf32_tflops_burst": 2 * n ** 3 / best / 1e12, "tf32_tflops_sustained": sus,
                      "how": "torch.matmul fp32 with allow_tf32, 8192^3"}))


if __name__ == "__main__":
    main()
