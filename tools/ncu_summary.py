"""Summarise ncu outputs for profiles/: a launch list CSV (per-kernel share of
device time) and/or an ncu-rep capture (key roofline counters).

usage: python tools/ncu_summary.py launches <launches.csv> [out.txt]
       python tools/ncu_summary.py rep <capture.ncu-rep> [out.txt]
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "gpc__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "sm__sass_thread_inst_executed_op_fadd_pred_on.sum",
        "sm__sass_thread_inst_executed_op_fmul_pred_on.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        name = name.replace("void ", "").replace("gpk::", "").replace("<unnamed>::", "")[:70]
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[name] += 1
    T = sum(tot.values())
    out = io.StringIO()
    out.write(f"{'us total':>12} {'share':>6} {'launches':>8} {'us/launch':>10}  kernel\n")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.write(f"{v:12.1f} {100 * v / T:5.1f}% {cnt[k]:8d} {v / cnt[k]:10.2f}  {k}\n")
    out.write(f"total {T:.1f} us over {sum(cnt.values())} launches (ncu serialised, cold caches)\n")
    return out.getvalue()


def rep(path):
    csvtext = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(csvtext)))
    h, units = rows[0], rows[1]
    out = io.StringIO()
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        out.write(f"kernel: {name[:120]}\n")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                out.write(f"  {k:66s} {r[i]:>18s} {units[i]}\n")
    return out.getvalue()


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    text = launches(path) if mode == "launches" else rep(path)
    if len(sys.argv) > 3:
        open(sys.argv[3], "w").write(text)
    print(text)
