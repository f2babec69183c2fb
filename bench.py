"""Benchmark of the matrix-free GP operator hot path (arXiv 2405.18457).

Default arm (ours): BASELINE.json config C2 (n=16384, d=26, alternating
projections b=512, s=64 pathwise probes, 2048 random features = 1024 sin/cos
pairs, warm start, tau=0.01, Adam lr 0.1) on synthetic sin-sum data. A "step"
is one marginal-likelihood step: RFF pathwise targets -> warm-started AP solve
of the n x 65 system -> fused gradient pass -> Adam, all device-resident.

  value       K.V kernel evals x RHS per second over the timed steps (evals
              counted on the device by every executed operator launch), with
              the dataset and solver state resident in HBM; L2 is flushed
              (256 MiB write) between timed steps.
  e2e         the same metric through the public C-ABI call gpk_optimise on
              host buffers (dataset H2D and trace D2H inside the timed region).
  roofline    fused K.V kernels (the persistent AP solver and kv_tc_kernel):
              achieved = the algorithmic FP32 flops of SURVEY 8d, F_KV =
              2m + 3d + 6 per executed kernel entry (counted on the device) /
              summed CUDA-event launch time, against the FP32 SIMT peak 148 SM x
              128 lanes x 2 x measured SM clock (the north star's "FP32
              compute roofline"). The kernels move the 2m contraction flops
              (and, for d >= 16, the distance Gram terms) onto the tcgen05
              tensor cores, so frac can exceed what FP32 FMA alone could do;
              the FP32-pipe share (3d + 6 per entry: distance, sqrt, exp) is
              reported beside it as fp32_pipe_tflops / fp32_pipe_frac.
  cpu_baseline the FP64 oracle (restated reference, C++) on the host cores,
              one H.V row slab per sample.

--impl reference times the reference's CPU implementation of the same path
(the FP64 restatement in oracle/, since the reference itself cannot be built
here: Eigen3 is absent) on all host threads.

Multi-GPU (torchrun, N > 1): C2 is a single-GPU configuration, so each rank
runs an independent replica (weak scaling); value = all ranks' evals / the
slowest rank's time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "K.V kernel evals x RHS per second"
UNIT = "evals*rhs/s"

CONFIGS = {
    "C1": dict(n=4096, d=8, uniform=False, noise=0.1, kind=0, s=16, rff_pairs=512, steps=10, max_epochs=50,
               block=1000, batch=500, lr_sgd=30.0),
    "C2": dict(n=16384, d=26, uniform=False, noise=0.1, kind=1, s=64, rff_pairs=1024, steps=20, max_epochs=50,
               block=512, batch=500, lr_sgd=30.0),
    "C3": dict(n=43008, d=20, uniform=False, noise=0.1, kind=0, s=64, rff_pairs=1000, steps=50, max_epochs=10,
               block=1000, batch=500, lr_sgd=30.0),
    "C4": dict(n=393216, d=3, uniform=True, noise=0.05, kind=2, s=64, rff_pairs=1000, steps=30, max_epochs=10,
               block=1000, batch=512, lr_sgd=10.0),
    "C5": dict(n=1835008, d=11, uniform=False, noise=0.1, kind=0, s=64, rff_pairs=2048, steps=15, max_epochs=5,
               block=1000, batch=500, lr_sgd=30.0),
}
WORKLOAD = "C2"
SEEDS = dict(data=0, probe=2, feature=3, solver=4)


def workload_config(name):
    c = CONFIGS[name]
    desc = {"C1": "CG", "C2": "AP b=512", "C3": "CG T=10", "C4": "SGD b=512 momentum 0.9", "C5": "CG T=5"}[name]
    return {"workload": f"{name}: n={c['n']} d={c['d']} {desc} s={c['s']} rff_pairs={c['rff_pairs']} "
                        f"warm start tol 0.01 Adam lr 0.1 (BASELINE.json configs[{list(CONFIGS).index(name)}])",
            "n": c["n"], "d": c["d"], "rhs": c["s"] + 1, "solver": desc, "l2": "flushed between timed steps",
            "data": "synthetic sin-sum (BASELINE.json generator, seed 0)"}


def init_constrained(c):
    """BASELINE.json: Matérn-3/2 ARD init lengthscales 1, signal 1, noise 0.1."""
    return [1.0] * c["d"] + [1.0, 0.1]


def outer_config(G, name, steps):
    c = CONFIGS[name]
    sc = G.SolverConfig(kind=c["kind"], tolerance=0.01, max_epochs=c["max_epochs"], block_size=c["block"],
                        batch_size=c["batch"], learning_rate=c["lr_sgd"], momentum=0.9, preconditioner_rank=100)
    return G.OuterConfig(estimator=1, solver=sc, warm_start=True, steps=steps, learning_rate=0.1,
                         probe_count=c["s"], rff_pairs=c["rff_pairs"], probe_seed=SEEDS["probe"],
                         feature_seed=SEEDS["feature"], solver_seed=SEEDS["solver"])


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML
    polled every 5 ms from a thread (nvidia-smi -lms 100 as the fallback)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._proc = None
        self._thread = None
        self._nvml = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._nvml = pynvml

            def poll():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    except Exception:
                        break
                    self.rows.append((float(sm), float(mx), int(bits)))
                    time.sleep(0.005)

            self._thread = threading.Thread(target=poll, daemon=True)
            self._thread.start()
            return
        except Exception:
            self._nvml = None
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                           "--format=csv,noheader,nounits", "-lms", "100"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self._proc = None

    def _read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self._proc.stdout:
            if self._stop.is_set():
                break
            r = [x.strip() for x in line.split(",")]
            try:
                bits = 0
                for k, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        bits |= self.REASONS[k]
                self.rows.append((float(r[1]), float(r[2]), bits))
            except (ValueError, IndexError):
                continue

    def stop(self):
        self._stop.set()
        if self._thread:
            self._thread.join(timeout=1)
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()

    def summary(self):
        sm = [r[0] for r in self.rows]
        mx = [r[1] for r in self.rows]
        reasons = sorted({k for r in self.rows for k, b in self.REASONS.items() if r[2] & b})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm), "source": "nvml 5 ms" if self._nvml else "nvidia-smi 100 ms"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(backend="nccl" if os.environ.get("GPK_BENCH_BACKEND", "nccl") == "nccl" else "gloo")
    return world, rank, local


def allreduce_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_slab_rate(name, threads, target_seconds, rows=256, reps_min=2):
    """Oracle (FP64 restated reference) H.V on a row slab of the workload."""
    from oracle import oracle as O
    c = CONFIGS[name]
    X32, _ = O.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], SEEDS["data"])
    X = np.asfortranarray(X32.astype(np.float64))
    m = c["s"] + 1
    raw = O.raw_from_constrained([1.0] * c["d"] + [1.0, 0.1])
    V = np.asfortranarray(np.random.default_rng(0).standard_normal((c["n"], m)))
    idx = np.arange(rows, dtype=np.int32)
    times = []
    t_start = time.perf_counter()
    while len(times) < reps_min or time.perf_counter() - t_start < target_seconds:
        t0 = time.perf_counter()
        O.apply_rows(X, raw, idx, V, threads=threads)
        times.append(time.perf_counter() - t0)
        if len(times) > 1000:
            break
    per = rows * c["n"] * m
    return per / float(np.mean(times)), len(times), float(np.sum(times))


def run_reference(args, world, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    c = CONFIGS[WORKLOAD]
    from oracle import oracle as O
    O.lib()
    rows = 256
    X32, _ = O.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], SEEDS["data"])
    X = np.asfortranarray(X32.astype(np.float64))
    m = c["s"] + 1
    raw = O.raw_from_constrained([1.0] * c["d"] + [1.0, 0.1])
    V = np.asfortranarray(np.random.default_rng(0).standard_normal((c["n"], m)))
    idx = np.arange(rows, dtype=np.int32)
    for _ in range(args.warmup):
        O.apply_rows(X, raw, idx, V, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.apply_rows(X, raw, idx, V, threads=threads)
    dt = time.perf_counter() - t0
    value = args.steps * rows * c["n"] * m / dt
    sample = f"{rows}-row slab of H.V at {WORKLOAD} (n={c['n']}, d={c['d']}, m={m}) per step, FP64"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(WORKLOAD),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference = FP64 C++ restatement of proj/core/src (oracle/); the reference itself needs "
                    "Eigen3, absent here"}
    print(json.dumps(line), flush=True)


def l2_flush(buf):
    buf.add_(1.0)


def run_ours(args, world, rank, local):
    import torch

    import paper_2405_18457_b200 as G

    torch.cuda.set_device(local)
    c = CONFIGS[WORKLOAD]
    ctx = G.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=local)
    X32, y32 = G.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], SEEDS["data"])
    X, y = X32.astype(np.float64), y32.astype(np.float64)
    total_steps = args.warmup + args.steps
    opt = G.Optimiser(ctx, X, y, outer_config(G, WORKLOAD, total_steps), init_constrained=init_constrained(c))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2
    opt.step(args.warmup)
    ctx.synchronize()
    ctx.reset_stats()
    ctx.set_profiling(True)
    launches0 = ctx.launch_count()
    clocks = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    evs = []
    traces = []
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            traces.append(opt.step(1))
            e1.record(stream)
            evs.append((e0, e1))
    torch.cuda.synchronize()
    barrier(world)
    clocks.stop()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    st = ctx.stats()
    launches = ctx.launch_count() - launches0
    ctx.set_profiling(False)
    ms_max = allreduce_max(ms, world)
    evals_total = allreduce_sum(st["evals_x_rhs"], world)
    value = evals_total / (ms_max / 1e3)
    clk = clocks.summary()
    f_sm = (clk["sm_mhz"] or 1965.0) * 1e6
    peak = 148 * 128 * 2 * f_sm / 1e12
    achieved = st["flops"] / (st["kv_ms"] / 1e3) / 1e12 if st["kv_ms"] > 0 else None
    fp32_pipe = st["fp32_pipe_flops"] / (st["kv_ms"] / 1e3) / 1e12 if st["kv_ms"] > 0 else None
    iters = [int(t["iterations"][0]) for t in traces]
    epochs = [float(t["epochs"][0]) for t in traces]
    traffic = None
    prof_json = os.path.join(ROOT, "profiles", f"ncu_{WORKLOAD}_kv_traffic.json")
    if os.path.exists(prof_json):
        try:
            traffic = json.load(open(prof_json)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    opt.close()  # the device-timed job is finished; its buffers return to the device pool
    # ---- e2e: public C-ABI call on host buffers (dataset H2D + trace D2H inside) ----
    ctx.reset_stats()
    ecfg = outer_config(G, WORKLOAD, args.steps)
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eopt = G.Optimiser(ctx, X, y, ecfg, init_constrained=init_constrained(c))  # dataset H2D
    t1 = time.perf_counter()
    res = eopt.step(args.steps)  # trace D2H per step
    t2 = time.perf_counter()
    eopt.close()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    e2e_s = allreduce_max(t3 - t0, world)
    e2e_parts = {"create_s": t1 - t0, "steps_s": t2 - t1, "close_s": t3 - t2}
    e2e_evals = allreduce_sum(ctx.stats()["evals_x_rhs"], world)
    e2e_value = e2e_evals / e2e_s
    h2d = (X.nbytes + y.nbytes) / args.steps
    d2h = (2 * (c["d"] + 2) + 8) * 8

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, reps, secs = cpu_slab_rate(WORKLOAD, threads, args.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{reps} x 256-row H.V slabs of {WORKLOAD} (FP64 oracle, {secs:.1f} s)"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32 operator / f64 solver", "data": "synthetic",
                "config": dict(workload_config(WORKLOAD),
                               parallelism="replicas" if world > 1 else "single-gpu"),
                "seconds_per_ml_step": ms_max / args.steps / 1e3,
                "solver_iterations_per_step": iters, "epochs_per_step": epochs,
                "roofline": {"bound": "fp32_simt", "kernel": "ap_persistent_kernel + kv_tc_kernel (tcgen05 3xTF32)",
                             "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                             "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                             "peak_source": "148 SM x 128 FP32 lanes x 2 x median SM clock under load "
                                            "(MEASURED_PEAKS.json holds no FP32 SIMT figure)",
                             "achieved_counts": "SURVEY 8d algorithmic flops F_KV = 2m+3d+6 per executed kernel "
                                                "entry (the 2m contraction runs on tcgen05)",
                             "fp32_pipe_tflops": fp32_pipe,
                             "fp32_pipe_frac": (fp32_pipe / peak) if fp32_pipe else None,
                             "kv_launches": st["kv_launches"], "kv_ms": st["kv_ms"],
                             "kv_share_of_step": st["kv_ms"] / ms if ms > 0 else None},
                "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "call": "gpk_optimiser_create/step/destroy (host buffers)",
                        "steps": int(len(res["iterations"])),
                        "seconds": e2e_s, "parts": e2e_parts,
                        "step_seconds": [round(float(v), 6) for v in res["step_seconds"]]},
                "gpu_launches": launches, "clocks": clk}
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)  # timing rule: at least 3 untimed warm-up steps
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
