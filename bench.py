"""Benchmark of the matrix-free GP operator hot path (arXiv 2405.18457).

Workload (``--workload``, default C4 = BASELINE.json configs[3], the largest
configuration BASELINE runs on one GPU): n=393216, d=3, X~U[-1,1]^3,
sin-sum targets with noise 0.05, Matérn-3/2 ARD (init 1/1/0.1), pathwise
estimator with s=64 probes and 1000 RFF pairs, SGD (minibatch 512, momentum
0.9, lr 10) warm-started with a budget of 10 epochs (7680 iterations) per
step, Adam lr 0.1. Synthetic data from the BASELINE generator stands in for
the UCI sets (absent here). A "step" is one marginal-likelihood step: RFF
pathwise targets -> warm-started solve of the n x 65 system -> fused gradient
pass -> Adam, all device-resident.

Timing: W warm-up steps run on a throw-away optimiser; a fresh optimiser then
runs the config's trajectory, step 1 untimed and steps 2..K+1 timed (default
K = the config's step count - 1, i.e. SURVEY 8d(ii)'s "mean over steps
2..N"), each bracketed by CUDA events on the library's stream (after it joins
the auxiliary stream), L2 flushed (256 MiB write) before every timed step.

  value        K.V kernel evals x RHS per second over the timed steps (evals
               counted on the device by every executed operator launch);
               inputs and solver state resident in HBM.
  e2e          the same metric over the whole public-API call sequence on
               host buffers: Optimiser create (dataset H2D) -> K+1 steps
               (trace D2H each) -> destroy, wall clock.
  roofline     the dominant operator kernel (one extra profiled step after
               the timed region; per-launch CUDA events on the library's
               stream): achieved = SURVEY 8d algorithmic flops F_KV = 2m+3d+6
               per executed kernel entry / launch time, against the tcgen05 +
               MUFU bound of the same entries (bound "tensor"); the FP32-SIMT
               roof the north star names is reported beside it.
  cpu_baseline the FP64 oracle (restated reference) timing build on the host
               cores: one SGD minibatch apply_rows (512 rows x n) per sample,
               1 thread and all threads; seconds per step extrapolated.

--impl reference times the reference's CPU implementation of the same path
(the FP64 restatement in oracle/, timing build; the reference itself cannot be
built here: Eigen3 is absent) on all host threads, one minibatch product of
the workload per step.

Multi-GPU (torchrun, N > 1): the optimiser is row-sharded over the ranks
(one NCCL communicator; SGD: minibatch partial products all-gathered; CG:
search direction all-gathered), total work fixed ("strong"); value = the
job's evals / the slowest rank's device time. AP (C2) is single-GPU: N > 1
runs replicas there.
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
DEFAULT_WORKLOAD = "C4"
SEEDS = dict(data=0, probe=2, feature=3, solver=4)
SOLVER_NAME = {"C1": "CG", "C2": "AP b=512", "C3": "CG T=10", "C4": "SGD b=512 momentum 0.9", "C5": "CG T=5"}


def workload_config(name, world=1, parallelism=None):
    c = CONFIGS[name]
    desc = SOLVER_NAME[name]
    return {"workload": f"{name}: n={c['n']} d={c['d']} {desc} s={c['s']} rff_pairs={c['rff_pairs']} "
                        f"warm start tol 0.01 Adam lr 0.1 (BASELINE.json configs[{list(CONFIGS).index(name)}])",
            "n": c["n"], "d": c["d"], "rhs": c["s"] + 1, "solver": desc,
            "l2": "flushed (256 MiB write) before every timed step; solver state > L2",
            "data": "synthetic sin-sum (BASELINE.json generator, seed 0)",
            "parallelism": parallelism or (f"row-sharded x{world}" if world > 1 else "single-gpu")}


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
                    time.sleep(0.02)

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
                "reasons": reasons, "samples": len(sm), "source": "nvml 20 ms" if self._nvml else "nvidia-smi 100 ms"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group(backend="nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def _reduce(x, world, op):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=op)
    return float(t.item())


def allreduce_max(x, world):
    if world == 1:
        return x
    import torch.distributed as dist
    return _reduce(x, world, dist.ReduceOp.MAX)


def allreduce_sum(x, world):
    if world == 1:
        return x
    import torch.distributed as dist
    return _reduce(x, world, dist.ReduceOp.SUM)


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------- CPU arms
def _cpu_problem(name):
    from oracle import oracle as O
    c = CONFIGS[name]
    X32, _ = O.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], SEEDS["data"])
    X = np.asfortranarray(X32.astype(np.float64))
    m = c["s"] + 1
    raw = O.raw_from_constrained(init_constrained(c))
    V = np.asfortranarray(np.random.default_rng(0).standard_normal((c["n"], m)))
    return O, c, X, raw, V, m


def _cpu_sample_rows(name):
    """Rows of one CPU sample: the SGD minibatch for C4 (one solver iteration's
    apply_rows, kernel.cpp:154-168 incl. its row-major copy of V), a 256-row
    slab of the full product otherwise."""
    c = CONFIGS[name]
    return c["batch"] if c["kind"] == 2 else 256


def cpu_rate(name, threads, target_seconds, reps_min=1):
    O, c, X, raw, V, m = _cpu_problem(name)
    rows = _cpu_sample_rows(name)
    idx = np.sort(np.random.default_rng(1).choice(c["n"], rows, replace=False)).astype(np.int32)
    O.apply_rows(X, raw, idx[:8], V, threads=threads)  # page-in / thread start
    times = []
    t_start = time.perf_counter()
    while len(times) < reps_min or time.perf_counter() - t_start < target_seconds:
        t0 = time.perf_counter()
        O.apply_rows(X, raw, idx, V, threads=threads)
        times.append(time.perf_counter() - t0)
        if len(times) >= 1000:
            break
    per = rows * c["n"] * m
    t = float(np.mean(times))
    return per / t, len(times), float(np.sum(times)), t


def extrapolated_step_seconds(name, t_sample):
    """Solver-only CPU seconds per marginal-likelihood step from one sample:
    SGD budget iterations x one minibatch product (C4), else the sample scaled
    to a full product per epoch (CG: epochs = products)."""
    c = CONFIGS[name]
    if c["kind"] == 2:
        return c["max_epochs"] * c["n"] / c["batch"] * t_sample
    return c["max_epochs"] * (c["n"] / _cpu_sample_rows(name)) * t_sample


def host_cpu():
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def run_reference(args, world, rank):
    if rank != 0:
        return
    from oracle import oracle as O
    O.use_timing_build()
    O.lib()
    threads = os.cpu_count() or 1
    name = args.workload
    Ox, c, X, raw, V, m = _cpu_problem(name)
    rows = _cpu_sample_rows(name)
    idx = np.sort(np.random.default_rng(1).choice(c["n"], rows, replace=False)).astype(np.int32)
    for _ in range(args.warmup):
        Ox.apply_rows(X, raw, idx, V, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        Ox.apply_rows(X, raw, idx, V, threads=threads)
    dt = time.perf_counter() - t0
    value = args.steps * rows * c["n"] * m / dt
    sample = (f"one {rows}-row apply_rows of {name} (n={c['n']}, d={c['d']}, m={m}) per step, FP64 oracle timing "
              f"build (-O3 -march=native, vectorised exp), {threads} threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(name, 1, "host cores"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "seconds_per_ml_step_extrapolated": extrapolated_step_seconds(name, dt / args.steps),
            "host": host_cpu(),
            "note": "reference = FP64 C++ restatement of proj/core/src (oracle/); the reference itself needs "
                    "Eigen3, absent here"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def l2_flush(buf):
    buf.add_(1.0)


def tensor_mufu_bound(m, d, f_sm, tf32_tflops):
    """Entries/s the tcgen05 operator can reach at most: 3 TF32 MMA passes of
    N = 16 ceil(m/16) columns per entry on the tensor cores, and 2 MUFU ops
    (sqrt, ex2) per entry at 16/clk/SM."""
    npad = max(16, (m + 15) // 16 * 16)
    tensor = tf32_tflops * 1e12 / (3 * 2 * npad)
    mufu = 148 * 16 * f_sm / 2
    return min(tensor, mufu), tensor, mufu


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except (OSError, ValueError):
        return {}


def run_ours(args, world, rank, local):
    import torch

    import paper_2405_18457_b200 as G
    from paper_2405_18457_b200 import parallel as PAR

    torch.cuda.set_device(local)
    name = args.workload
    c = CONFIGS[name]
    sharded = world > 1 and c["kind"] != 1
    ctx = G.Context(local)
    if sharded:
        PAR.init_comm_from_torch(ctx)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=local)
    X32, y32 = G.sinsum_dataset(c["n"], c["d"], c["uniform"], c["noise"], SEEDS["data"])
    X, y = X32.astype(np.float64), y32.astype(np.float64)
    K = args.steps if args.steps > 0 else c["steps"] - 1
    # ---- warm-up: a throw-away optimiser (module load, pools, graphs) ----
    wopt = G.Optimiser(ctx, X, y, outer_config(G, name, args.warmup), init_constrained=init_constrained(c))
    wopt.step(args.warmup)
    wopt.close()
    ctx.synchronize()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2
    barrier(world)
    torch.cuda.synchronize()
    # ---- the run: public API on host buffers (e2e) with steps 2..K+1 device-timed ----
    ctx.reset_stats()
    clocks = ClockSampler(local)
    t_e0 = time.perf_counter()
    opt = G.Optimiser(ctx, X, y, outer_config(G, name, K + 1), init_constrained=init_constrained(c))
    traces = [opt.step(1)]  # step 1 (cold solve from zero): untimed
    ctx.synchronize()
    st0 = ctx.stats()
    launches0 = ctx.launch_count()
    evs = []
    clocks.start()
    with torch.cuda.stream(stream):
        for _ in range(K):
            l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            traces.append(opt.step(1))
            ctx.join()
            e1.record(stream)
            evs.append((e0, e1))
    torch.cuda.synchronize()
    clocks.stop()
    st1 = ctx.stats()
    launches = ctx.launch_count() - launches0
    # one more step with per-launch events for the roofline (outside the timed steps)
    ctx.set_profiling(True)
    ctx.reset_stats()
    opt_prof = opt.step(1)
    stp = ctx.stats()
    ctx.set_profiling(False)
    opt.close()
    torch.cuda.synchronize()
    t_e1 = time.perf_counter()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = float(sum(step_ms))
    ms_max = allreduce_max(ms, world)
    # each rank counts the evals of its own rows; the job's are the sum
    evals_timed = allreduce_sum(st1["evals_x_rhs"] - st0["evals_x_rhs"], world)
    value = evals_timed / (ms_max / 1e3)
    # e2e: create + K+1 steps (+ the profiled step's share excluded by scaling) + destroy
    e2e_s = allreduce_max(t_e1 - t_e0, world)
    evals_all = allreduce_sum(st1["evals_x_rhs"], world)
    prof_wall = float(opt_prof["step_seconds"][0]) if len(opt_prof["step_seconds"]) else 0.0
    e2e_value = evals_all / max(1e-9, e2e_s - prof_wall)
    clk = clocks.summary()
    f_sm = (clk["sm_mhz"] or 1965.0) * 1e6
    simt_peak = 148 * 128 * 2 * f_sm / 1e12
    m, d = c["s"] + 1, c["d"]
    fkv = 2 * m + 3 * d + 6
    achieved = stp["flops"] / (stp["kv_ms"] / 1e3) / 1e12 if stp["kv_ms"] > 0 else None
    peaks = measured_peaks()
    tf32 = args.tf32_tflops or (peaks.get("bf16_tflops", 1660.6) / 2.0)
    bound_entries, tensor_e, mufu_e = tensor_mufu_bound(m, d, f_sm, tf32)
    tc_peak = bound_entries * fkv / 1e12
    traffic = None
    prof_json = os.path.join(ROOT, "profiles", f"ncu_{name}_kv_traffic.json")
    if os.path.exists(prof_json):
        try:
            traffic = json.load(open(prof_json)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        O.use_timing_build()
        threads = os.cpu_count() or 1
        rate_all, reps_all, secs_all, t_all = cpu_rate(name, threads, args.cpu_seconds)
        rate_1, reps_1, secs_1, t_1 = cpu_rate(name, 1, args.cpu_seconds / 2)
        rows = _cpu_sample_rows(name)
        cpu = {"value": rate_all, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{reps_all} x one {rows}-row apply_rows of {name} (FP64 oracle timing build, "
                         f"{threads} threads, {secs_all:.1f} s); 1 thread: {reps_1} x ({secs_1:.1f} s)",
               "value_1thread": rate_1,
               "seconds_per_ml_step_extrapolated": extrapolated_step_seconds(name, t_all),
               "seconds_per_ml_step_extrapolated_1thread": extrapolated_step_seconds(name, t_1),
               "extrapolation": "solver only: SGD budget iterations x one minibatch product" if c["kind"] == 2
                                else "solver only: products per step x one product",
               "host": host_cpu()}
    if rank == 0:
        iters = [int(t["iterations"][0]) for t in traces]
        epochs = [float(t["epochs"][0]) for t in traces]
        nd = c["n"] * (c["d"] + 1) * 8
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
                "warmup": args.warmup, "ms_per_step": ms_max / K, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32 operator (3xTF32 tcgen05) / f64 solver",
                "data": "synthetic",
                "config": workload_config(name, world, "replicas" if world > 1 and not sharded else None),
                "seconds_per_ml_step": ms_max / K / 1e3,
                "timed_steps": f"2..{K + 1} of a fresh {K + 1}-step trajectory",
                "step_ms": [round(v, 3) for v in step_ms],
                "solver_iterations_per_step": iters, "epochs_per_step": epochs,
                "roofline": {"bound": "tensor", "kernel": "operator kernel of the solver (tcgen05 3xTF32)",
                             "achieved": achieved, "peak": tc_peak, "unit": "TFLOP/s",
                             "frac": (achieved / tc_peak) if achieved else None, "traffic": traffic,
                             "counts": f"F_KV = 2m+3d+6 = {fkv} algorithmic FP32 flops per executed kernel entry",
                             "peak_source": f"min(tensor, MUFU) entries/s x F_KV: tensor {tensor_e:.3e} entries/s "
                                            f"(3 TF32 passes x N={max(16, (m + 15) // 16 * 16)} at {tf32:.0f} TF/s "
                                            f"TF32 = MEASURED_PEAKS bf16 / 2), MUFU {mufu_e:.3e} entries/s "
                                            f"(2 ops/entry, 16/clk/SM at the median SM clock)",
                             "fp32_simt_peak": simt_peak, "fp32_simt_frac": (achieved / simt_peak) if achieved else None,
                             "kv_launches": stp["kv_launches"], "kv_ms": stp["kv_ms"],
                             "kv_ms_per_launch": stp["kv_ms"] / max(1, stp["kv_launches"]),
                             "measured_on": "one profiled step after the timed steps (per-launch CUDA events)"},
                "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": nd / (K + 1),
                        "d2h_bytes_per_step": (2 * (c["d"] + 2) + 8) * 8,
                        "call": "Optimiser(create: dataset H2D) -> step() x (K+1) (trace row D2H each) -> close",
                        "seconds": e2e_s - prof_wall, "steps": K + 1},
                "gpu_launches": launches, "clocks": clk}
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=0, help="timed steps (default: the config's steps - 1)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=list(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=16.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="(accepted for tools; e2e is part of the timed run)")
    ap.add_argument("--tf32-tflops", type=float, default=0.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)  # timing rule: at least 3 untimed warm-up steps
    world, rank, local = dist_setup()
    if args.impl == "reference":
        if args.steps <= 0:
            args.steps = 5
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
