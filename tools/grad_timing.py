"""Times the fused gradient pass (pathwise pair set: v_y (1 column) and s
probe solutions) at BASELINE shapes, tensor-core (GPK_KERNEL=1, default) or
SIMT (GPK_KERNEL=0) gradient kernel. Device-synchronised wall time per call."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_18457_b200 as G  # noqa: E402


def main():
    ctx = G.Context(0)
    ctx.set_operator_kernel(int(os.environ.get("GPK_KERNEL", "1")))
    shapes = [(16384, 26, 64), (4096, 8, 16), (43008, 20, 64)]
    if len(sys.argv) == 4:
        shapes = [tuple(int(v) for v in sys.argv[1:4])]
    for n, d, s in shapes:
        rng = np.random.default_rng(0)
        X = rng.standard_normal((n, d))
        raw = np.array([G.gpiter.softplus_inverse(1.0)] * (d + 1) + [G.gpiter.softplus_inverse(0.1)])
        op = G.KernelOperator(X, G.Hyperparameters.from_raw(raw), ctx)
        vy = rng.standard_normal(n)
        Z = rng.standard_normal((n, s))
        G.estimate_gradient_pathwise(op, vy, Z)
        reps = 5
        ctx.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            G.estimate_gradient_pathwise(op, vy, Z)
        ctx.synchronize()
        dt = (time.perf_counter() - t) / reps
        pairs = n * (n + 1) / 2
        print(json.dumps({"n": n, "d": d, "s": s, "seconds_per_call": dt, "pairs_per_s": pairs / dt}), flush=True)


if __name__ == "__main__":
    main()
