"""Lists every GPU activity (kernel / copy) of one warm C2 optimiser step with
its stream, start offset and duration (CUPTI via torch.profiler), to read the
main/auxiliary stream overlap of the AP block inverses."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2405_18457_b200 as G  # noqa: E402


def main():
    name = "C2"
    c = bench.CONFIGS[name]
    ctx = G.Context(0)
    X32, y32 = G.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], bench.SEEDS["data"])
    X, y = X32.astype(np.float64), y32.astype(np.float64)
    opt = G.Optimiser(ctx, X, y, bench.outer_config(G, name, 6), init_constrained=bench.init_constrained(c))
    opt.step(4)
    ctx.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        opt.step(1)
        ctx.synchronize()
    path = "/tmp/step_trace.json"
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
    gpu.sort(key=lambda e: e["ts"])
    t0 = gpu[0]["ts"]
    for e in gpu:
        print(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f}  s{e.get('args', {}).get('stream', '?'):<4} {e['name'][:90]}")


if __name__ == "__main__":
    main()
