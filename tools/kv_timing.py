"""Times the fused K.V operator kernel (gpk_apply_device) at BASELINE shapes.
Device-resident FP32 RHS, FP64 output, CUDA events on the library's stream."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18457_b200 as G  # noqa: E402

PEAK_FP32 = 148 * 128 * 2 * 1.965e9  # FLOP/s at the 1965 MHz max clock


def time_apply(ctx, n, d, m, reps=5, warm=2):
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, d))
    raw = np.array([G.gpiter.softplus_inverse(1.0)] * d + [G.gpiter.softplus_inverse(1.0),
                                                            G.gpiter.softplus_inverse(0.1)])
    op = G.KernelOperator(X, G.Hyperparameters.from_raw(raw), ctx)
    ld = G.load().gpk_rhs_ld(m)
    v = torch.zeros((n, ld), dtype=torch.float32, device="cuda")
    v[:, :m] = torch.randn((n, m), device="cuda")
    out = torch.empty((n, m), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream())
    lib = G.load()
    for _ in range(warm):
        G._lib.check(lib.gpk_apply_device(op.handle, C.c_void_p(v.data_ptr()), m, C.c_void_p(out.data_ptr()), m))
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        G._lib.check(lib.gpk_apply_device(op.handle, C.c_void_p(v.data_ptr()), m, C.c_void_p(out.data_ptr()), m))
    e1.record(stream)
    e1.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    fkv = 2 * m + 3 * d + 6
    fpipe = 3 * d + 6 if os.environ.get("GPK_KERNEL", "1") == "1" else fkv  # FP32-pipe share (tcgen05 kernel)
    return {"n": n, "d": d, "m": m, "seconds": t, "evals_x_rhs_per_s": n * n * m / t,
            "fp32_equivalent_tflops": n * n * fkv / t / 1e12, "fp32_equivalent_frac": n * n * fkv / t / PEAK_FP32,
            "fp32_pipe_tflops": n * n * fpipe / t / 1e12, "fp32_pipe_frac": n * n * fpipe / t / PEAK_FP32}


if __name__ == "__main__":
    ctx = G.Context(0)
    kernel = int(os.environ.get("GPK_KERNEL", "1"))
    ctx.set_operator_kernel(kernel)
    shapes = [(4096, 8, 17), (16384, 26, 65), (43008, 20, 65), (131072, 3, 65), (131072, 11, 65)]
    if len(sys.argv) == 4:  # single shape: n d m
        shapes = [tuple(int(a) for a in sys.argv[1:4])]
    for n, d, m in shapes:
        r = time_apply(ctx, n, d, m)
        r["kernel"] = ["simt", "tcgen05"][kernel]
        print(json.dumps(r), flush=True)
