"""GPU timeline of warm C2 optimiser steps (bench.py's workload) from the
CUDA activity trace (torch.profiler / CUPTI sees every kernel and copy of the
process, libgpk's included): per-step busy time, idle gaps > 4 us with the
activities either side, and per-kernel totals.

usage: python tools/timeline.py [steps] [config]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2405_18457_b200 as G  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    name = sys.argv[2] if len(sys.argv) > 2 else "C2"
    c = bench.CONFIGS[name]
    ctx = G.Context(0)
    X32, y32 = G.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], bench.SEEDS["data"])
    X, y = X32.astype(np.float64), y32.astype(np.float64)
    opt = G.Optimiser(ctx, X, y, bench.outer_config(G, name, 3 + steps), init_constrained=bench.init_constrained(c))
    opt.step(3)
    ctx.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(steps):
            opt.step(1)
        ctx.synchronize()
    path = "/tmp/timeline_trace.json"
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
    gpu.sort(key=lambda e: e["ts"])
    t0, t1 = gpu[0]["ts"], max(e["ts"] + e["dur"] for e in gpu)
    # union of busy intervals
    busy, cur_s, cur_e = 0.0, None, None
    gaps = []
    last_name = None
    for e in gpu:
        s, d = e["ts"], e["ts"] + e["dur"]
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
                if s - cur_e > 4:
                    gaps.append((s - cur_e, last_name, e["name"]))
            cur_s, cur_e = s, d
        else:
            cur_e = max(cur_e, d)
        last_name = e["name"] if d >= cur_e else last_name
    busy += cur_e - cur_s
    span = t1 - t0
    print(json.dumps({"steps": steps, "span_us_per_step": span / steps, "busy_us_per_step": busy / steps,
                      "idle_us_per_step": (span - busy) / steps, "gaps_over_4us": len(gaps)}))
    agg = {}
    for g, a, b in gaps:
        k = (a[:50], b[:50])
        agg.setdefault(k, [0, 0.0])
        agg[k][0] += 1
        agg[k][1] += g
    for (a, b), (cnt, tot) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
        print(f"  gap {tot / steps:8.1f} us/step  x{cnt / steps:5.1f}  after {a}  ->  before {b}")
    kt = {}
    for e in gpu:
        k = e["name"][:60]
        kt.setdefault(k, [0, 0.0])
        kt[k][0] += 1
        kt[k][1] += e["dur"]
    for k, (cnt, tot) in sorted(kt.items(), key=lambda x: -x[1][1])[:25]:
        print(f"  kernel {tot / steps:8.1f} us/step  x{cnt / steps:6.1f}  {k}")


if __name__ == "__main__":
    main()
